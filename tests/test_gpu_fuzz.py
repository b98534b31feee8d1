"""Seeded randomized parity over the configuration space: pool size (including M not dividing
C, partial pools and pools smaller than a tile), d, batch sizes, world size (emulated shards),
K, scale and margin, and every NEXT-3 variant -- each case against the fp64 oracle with the BJ:5
tolerances.  The cases are fixed by their seeds, so a failure is reproducible by its id."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_loss_close, from_dev, lt, to_dev

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("F2C_FUZZ_CASES", "64"))  # (a longer sweep: F2C_FUZZ_CASES=512)
FIRST = int(os.environ.get("F2C_FUZZ_FIRST", "0"))  # first case index (sweeps beyond the default cases)


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _case(i):
    rng = np.random.default_rng(1000 + i)
    W = int(rng.choice([1, 1, 2, 3]))
    K = int(rng.choice([1, 1, 1, 2, 3]))
    d = int(rng.choice([128, 256, 384, 512]))
    C = int(rng.integers(max(W, 3), 2600))
    m_loc = int(rng.integers(1, max(2, min(96, C // W) + 1)))
    n_loc = int(rng.integers(1, 200))
    fill = float(rng.choice([0.3, 1.0, 2.5]))            # partial pool, just full, wrapped
    s = float(rng.choice([1.0, 30.0, 64.0, 100.0]))
    m = float(rng.choice([0.0, 0.2, 0.35]))
    phi_mode = int(rng.choice([oracle.PHI_MEAN, oracle.PHI_MEAN, oracle.PHI_SUM, oracle.PHI_MAX]))
    hinge = bool(rng.random() < 0.25)
    lam = float(rng.choice([1.0, 1.0, 0.5]))
    excl = bool(rng.random() < 0.25)
    refresh = bool(rng.random() < 0.2)
    n_lab = int(rng.integers(max(2, m_loc * W + 1), 4 * C + 10))
    # fp32 pools (tf32 logits, BJ:7 / D21) where they apply: K = 1, d <= 256
    dt = synth.F32 if (K == 1 and d <= 256 and rng.random() < 0.35) else synth.BF16
    if dt == synth.F32:
        # tf32 logits round the cosines by ~1e-4: a sum / mean hinge then has near-zero cosines on
        # both sides of 0 in most rows (D21); fp32 pools are fuzzed without the hinge
        hinge = False
    return dict(W=W, K=K, d=d, C=C, m_loc=m_loc, n_loc=n_loc, fill=fill, s=s, m=m, phi_mode=phi_mode,
                hinge=hinge, lam=lam, excl=excl, refresh=refresh, n_lab=n_lab, seed=2000 + i, dt=dt)


@pytest.mark.parametrize("i", range(FIRST, FIRST + N_CASES))
def test_fuzz_parity(dcp, i):
    c = _case(i)
    W, K, d, C, m_loc = c["W"], c["K"], c["d"], c["C"], c["m_loc"]
    dt = c["dt"]
    head = dcp.DCPHead(C, d, dt, world=W, rank=0 if W == 1 else -1, n_local_max=c["n_loc"],
                       m_local_max=m_loc, K=K)
    head.set_lcos(c["phi_mode"], c["hinge"], c["lam"])
    head.set_dup_mode(c["excl"])
    head.set_enqueue_mode(c["refresh"])
    pool = oracle.Pool(C, d, dt, K=K)
    rng = np.random.default_rng(c["seed"])
    Mg = m_loc * W
    nblk = max(1, int(c["fill"] * C / Mg))
    for b in range(nblk):
        G = synth.unit_rows(c["seed"], synth.S_PRE, b, 0, Mg * K, d, dt)
        if K > 1:  # arbitrary bf16 features, K per slot (NEXT-1: exact-mean logits)
            G = G.reshape(Mg, K, d)
        y = rng.choice(c["n_lab"], size=Mg, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, dt), lt(y))
        pool.enqueue(G, y, refresh=c["refresh"])
    N = c["n_loc"] * W
    X = synth.unit_rows(c["seed"] + 1, synth.S_INST, 0, 0, N, d, dt)
    occ = pool.C_occ
    y = rng.integers(0, c["n_lab"], N).astype(np.int64)
    y[::2] = pool.lab[:occ][rng.integers(0, occ, len(y[::2]))]
    if c["phi_mode"] == oracle.PHI_MAX:
        # hardest negatives far from ties: out-of-pool rows are noisy copies of pool centers
        neg = np.where(~np.isin(y, pool.lab[:occ]))[0]
        Tf = oracle.bf16_to_f64(pool.T) if dt == synth.BF16 else pool.T.astype(np.float64)
        Tb = Tf.reshape(C, K, d).mean(axis=1)
        v = Tb[rng.integers(0, occ, len(neg))] + 0.25 * rng.standard_normal((len(neg), d)) / np.sqrt(d)
        v = v / np.maximum(np.linalg.norm(v, axis=1, keepdims=True), 1e-12)
        X[neg] = oracle.f64_to_bf16(v) if dt == synth.BF16 else v.astype(np.float32)
    loss, dx = head.loss_fwd_bwd(to_dev(X, dt), lt(y), None, c["s"], c["m"])
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, c["s"], c["m"], phi_mode=c["phi_mode"], hinge=c["hinge"], lam=c["lam"],
                    excl_dup=c["excl"])
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0]), c
    np.testing.assert_array_equal(labs, pool.lab)
    assert_loss_close(float(loss.item()), ref.L, what=f"loss {c}")
    rows = np.arange(N)
    if c["hinge"]:
        # The hinge max(0, cos) is discontinuous at cos = 0: a pair whose cosine lies within the GPU's
        # rounding of 0 may be decided either way, and each decision moves that row's gradient by a
        # whole (weighted) center.  Both decisions are correct; such rows are compared through their
        # loss only (their phi terms differ by < the rounding), the rest element by element.  The logits
        # are fp32 accumulations of exact bf16 products (K d terms), accurate to ~1e-7.
        occ = pool.C_occ
        Tf = oracle.bf16_to_f64(pool.T) if dt == synth.BF16 else pool.T.astype(np.float64)
        Tb = Tf.reshape(C, K, d).mean(axis=1)[:occ]
        Xf = oracle.bf16_to_f64(X) if dt == synth.BF16 else X.astype(np.float64)
        xh = Xf / np.linalg.norm(Xf, axis=1, keepdims=True)
        neg = np.where(ref.tslot < 0)[0]
        tol = 2e-6 * np.linalg.norm(Tb, axis=1)   # (~20x the fp32-accumulation error of the logits)
        amb = (np.abs(xh[neg] @ Tb.T) < tol[None, :]).any(axis=1)
        # (a guard on the test's strength, not on parity: most rows must still be compared element by
        # element.  The expected count is ~ N_neg C_occ 1.6e-6 sqrt(d); case 1073 of the 3000-case sweep
        # has 8 such rows of 29 against 2 expected, so the cap is half the rows, not a quarter)
        assert amb.sum() <= max(3, 0.5 * len(neg)), (int(amb.sum()), len(neg), c)
        rows = np.setdiff1d(rows, neg[amb])
    assert_dx_close(from_dev(dx)[rows], ref.dx[rows], what=f"dx {c}")
