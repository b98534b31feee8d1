"""Seeded randomized parity at medium sizes: pools of 10K-60K slots (80-470 tiles: several
ranges per row group, multi-wave schedules at small cluster counts) and batches of up to 1600
rows (up to 13 row groups), against the fp64 oracle.  Each case costs the CPU oracle tens of
seconds, so the default run is one case; F2C_FUZZ_MED_CASES=16 for a sweep.  A third of the
cases also cap the fused kernel at 5 or 17 clusters (F2C_CLUSTERS: multi-wave schedules)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_loss_close, from_dev, lt, to_dev

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("F2C_FUZZ_MED_CASES", "1"))
FIRST = int(os.environ.get("F2C_FUZZ_FIRST", "0"))  # first case index (sweeps beyond the default cases)


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _case(i):
    rng = np.random.default_rng(90000 + i)
    W = int(rng.choice([1, 1, 2, 3]))
    K = int(rng.choice([1, 1, 1, 2, 3]))
    d = int(rng.choice([128, 256, 384, 512]))
    C = int(rng.integers(10000, 60000))
    m_loc = int(rng.integers(64, 1024)) // W
    n_loc = int(rng.integers(100, 1600)) // W
    fill = float(rng.choice([0.6, 1.0, 1.7]))            # partial pool, just full, wrapped
    s = float(rng.choice([1.0, 30.0, 64.0, 100.0]))
    m = float(rng.choice([0.0, 0.2, 0.35]))
    phi_mode = int(rng.choice([oracle.PHI_MEAN, oracle.PHI_MEAN, oracle.PHI_SUM, oracle.PHI_MAX]))
    hinge = bool(rng.random() < 0.25)
    lam = float(rng.choice([1.0, 1.0, 0.5]))
    excl = bool(rng.random() < 0.25)
    refresh = bool(rng.random() < 0.2)
    n_lab = int(rng.integers(max(2, m_loc * W + 1), 4 * C + 10))
    clusters = int(rng.choice([0, 0, 5, 17]))
    return dict(W=W, K=K, d=d, C=C, m_loc=m_loc, n_loc=n_loc, fill=fill, s=s, m=m, phi_mode=phi_mode,
                hinge=hinge, lam=lam, excl=excl, refresh=refresh, n_lab=n_lab, seed=92000 + i, clusters=clusters)


@pytest.mark.parametrize("i", range(FIRST, FIRST + N_CASES))
def test_fuzz_medium_parity(dcp, i, monkeypatch):
    c = _case(i)
    if c["clusters"]:
        monkeypatch.setenv("F2C_CLUSTERS", str(c["clusters"]))
    W, K, d, C, m_loc = c["W"], c["K"], c["d"], c["C"], c["m_loc"]
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=c["n_loc"],
                       m_local_max=m_loc, K=K)
    head.set_lcos(c["phi_mode"], c["hinge"], c["lam"])
    head.set_dup_mode(c["excl"])
    head.set_enqueue_mode(c["refresh"])
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    rng = np.random.default_rng(c["seed"])
    Mg = m_loc * W
    nblk = max(1, int(c["fill"] * C / Mg))
    for b in range(nblk):
        G = synth.unit_rows(c["seed"], synth.S_PRE, b, 0, Mg * K, d)
        if K > 1:  # arbitrary bf16 features, K per slot (NEXT-1: exact-mean logits)
            G = G.reshape(Mg, K, d)
        y = rng.choice(c["n_lab"], size=Mg, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=c["refresh"])
    N = c["n_loc"] * W
    X = synth.unit_rows(c["seed"] + 1, synth.S_INST, 0, 0, N, d)
    occ = pool.C_occ
    y = rng.integers(0, c["n_lab"], N).astype(np.int64)
    y[::2] = pool.lab[:occ][rng.integers(0, occ, len(y[::2]))]
    if c["phi_mode"] == oracle.PHI_MAX:
        # hardest negatives far from ties: out-of-pool rows are noisy copies of pool centers
        neg = np.where(~np.isin(y, pool.lab[:occ]))[0]
        Tb = oracle.bf16_to_f64(pool.T).reshape(C, K, d).mean(axis=1)
        v = Tb[rng.integers(0, occ, len(neg))] + 0.25 * rng.standard_normal((len(neg), d)) / np.sqrt(d)
        X[neg] = oracle.f64_to_bf16(v / np.maximum(np.linalg.norm(v, axis=1, keepdims=True), 1e-12))
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, c["s"], c["m"])
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, c["s"], c["m"], phi_mode=c["phi_mode"], hinge=c["hinge"], lam=c["lam"],
                    excl_dup=c["excl"])
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0]), c
    np.testing.assert_array_equal(labs, pool.lab)
    assert_loss_close(float(loss.item()), ref.L, what=f"loss {c}")
    assert_dx_close(from_dev(dx), ref.dx, what=f"dx {c}")
