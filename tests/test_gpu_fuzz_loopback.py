"""Seeded random configurations through the real per-rank multi-rank code path (the loopback transport,
tests/test_gpu_loopback.py): world 2-5, K in {1, 2}, bf16 or fp32 pools, every NEXT-3 variant, partial /
full / wrapped pools, ragged shards; several steps of enqueue + loss per case against the single-pool
oracle on the rank-ordered concatenation (D16).  F2C_FUZZ_LB_CASES sets the count (default 24)."""
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_loss_close, from_dev, it, lt, to_dev
from test_gpu_loopback import _loopback, _run_ranks

pytestmark = pytest.mark.gpu
N_CASES = int(os.environ.get("F2C_FUZZ_LB_CASES", "24"))
FIRST = int(os.environ.get("F2C_FUZZ_FIRST", "0"))  # first case index (sweeps beyond the default cases)


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _case(i):
    rng = np.random.default_rng(5000 + i)
    W = int(rng.integers(2, 6))
    K = int(rng.choice([1, 1, 2]))
    d = int(rng.choice([128, 256, 512]))
    dt = synth.F32 if (K == 1 and d <= 256 and rng.random() < 0.3) else synth.BF16
    C = int(rng.integers(W * 40, 3000))
    m_loc = int(rng.integers(1, max(2, min(64, C // W) + 1)))
    n_loc = int(rng.integers(1, 96))
    fill = float(rng.choice([0.4, 1.0, 2.5]))
    phi_mode = int(rng.choice([oracle.PHI_MEAN, oracle.PHI_MEAN, oracle.PHI_SUM, oracle.PHI_MAX]))
    hinge = bool(rng.random() < 0.3) and phi_mode == oracle.PHI_MAX   # (max + hinge: no near-zero flips)
    excl = bool(rng.random() < 0.25)
    refresh = bool(rng.random() < 0.25)
    n_lab = int(rng.integers(max(2, m_loc * W + 1), 3 * C + 10))
    return dict(W=W, K=K, d=d, dt=dt, C=C, m_loc=m_loc, n_loc=n_loc, fill=fill, phi_mode=phi_mode, hinge=hinge,
                excl=excl, refresh=refresh, n_lab=n_lab, seed=6000 + i, s=float(rng.choice([30.0, 64.0])),
                m=float(rng.choice([0.0, 0.35])))


@pytest.mark.parametrize("i", range(FIRST, FIRST + N_CASES))
def test_fuzz_loopback(dcp, monkeypatch, i):
    c = _case(i)
    W, K, d, dt, C, m_loc, n_loc = c["W"], c["K"], c["d"], c["dt"], c["C"], c["m_loc"], c["n_loc"]
    uid = _loopback(monkeypatch)
    rng = np.random.default_rng(c["seed"])
    Mg = m_loc * W
    nblk = max(1, int(c["fill"] * C / Mg))
    blocks = []
    for b in range(nblk + 2):
        G = synth.unit_rows(c["seed"], synth.S_PRE, b, 0, Mg * K, d, dt)
        if K > 1:
            G = G.reshape(Mg, K, d)
        y = rng.choice(c["n_lab"], size=Mg, replace=False).astype(np.int64)
        blocks.append((G, y))
    # the oracle first: each step's batch (and, for the hardest-negative variant, out-of-pool rows that
    # are noisy copies of pool centers, so the maximum is unique by a wide margin) and its result
    kw = dict(phi_mode=c["phi_mode"], hinge=c["hinge"], excl_dup=c["excl"])
    pool = oracle.Pool(C, d, dt, K=K)
    for G, y in blocks[:nblk]:
        pool.enqueue(G, y, refresh=c["refresh"])
    steps, refs = [], []
    for t in range(2):
        G, yb = blocks[nblk + t]
        pool.enqueue(G, yb, refresh=c["refresh"])
        X = synth.unit_rows(c["seed"] + 1, synth.S_INST, t, 0, W * n_loc, d, dt)
        y = rng.integers(0, c["n_lab"], W * n_loc).astype(np.int64)
        occ = pool.C_occ
        y[::3] = pool.lab[:occ][rng.integers(0, occ, len(y[::3]))]
        if c["phi_mode"] == oracle.PHI_MAX:
            neg = np.where(~np.isin(y, pool.lab[:occ]))[0]
            Tf = oracle.bf16_to_f64(pool.T) if dt == synth.BF16 else pool.T.astype(np.float64)
            Tb = Tf.reshape(C, K, d).mean(axis=1)
            v = Tb[rng.integers(0, occ, len(neg))] + 0.25 * rng.standard_normal((len(neg), d)) / np.sqrt(d)
            v = v / np.maximum(np.linalg.norm(v, axis=1, keepdims=True), 1e-12)
            X[neg] = oracle.f64_to_bf16(v) if dt == synth.BF16 else v.astype(np.float32)
        steps.append((X, y))
        refs.append(pool.loss(X, y, None, c["s"], c["m"], **kw))

    def rank_fn(r):
        head = dcp.DCPHead(C, d, dt, W, r, n_local_max=n_loc, m_local_max=m_loc, nccl_uid=uid, K=K)
        head.set_lcos(c["phi_mode"], c["hinge"], 1.0)
        head.set_dup_mode(c["excl"])
        head.set_enqueue_mode(c["refresh"])
        for G, y in blocks[:nblk]:
            head.enqueue(to_dev(G[r * m_loc:(r + 1) * m_loc], dt), lt(y[r * m_loc:(r + 1) * m_loc]))
        res = []
        for t, (X, y) in enumerate(steps):
            G, yb = blocks[nblk + t]
            head.enqueue(to_dev(G[r * m_loc:(r + 1) * m_loc], dt), lt(yb[r * m_loc:(r + 1) * m_loc]))
            loss, dx = head.loss_fwd_bwd(to_dev(X[r * n_loc:(r + 1) * n_loc], dt), lt(y[r * n_loc:(r + 1) * n_loc]),
                                         None, c["s"], c["m"])
            torch.cuda.current_stream().synchronize()
            res.append((float(loss.item()), from_dev(dx)))
        head.check()
        feats, labs, E = head.get_state()
        head.close()
        return res, labs, E

    out = _run_ranks(W, rank_fn)
    for t, ref in enumerate(refs):
        losses = [out[r][0][t][0] for r in range(W)]
        assert all(v == losses[0] for v in losses), (losses, c)
        assert_loss_close(losses[0], ref.L, what=f"loss {c}")
        assert_dx_close(np.concatenate([out[r][0][t][1] for r in range(W)]), ref.dx, what=f"dx {c}")
    np.testing.assert_array_equal(np.concatenate([o[1] for o in out]), pool.lab)
    assert all(o[2] == int(pool.E[0]) for o in out)
