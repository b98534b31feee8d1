"""The real multi-rank code path on one GPU: W handles, one per rank, each with its
own state buffer, host thread and stream, joined by the library's loopback test transport
(F2C_LOOPBACK=1: every NCCL collective of the protocol -- C1 all-gathers, C2 / refresh MAX all-reduces,
C3 all-gather, C4 reduce-scatter, C5 grouped send / recv of the routing plan -- executed as device
copies between the ranks' buffers, ordered by events).  Unlike the emulated world (one handle holding
every shard), this runs rank != 0 shards and buffers, the C5 plan's point-to-point pieces and the split
of the reduce-scatter through the same host code as NCCL.  Results must equal the single-pool oracle on
the rank-ordered concatenation (D16, pin P9); every rank must report the same loss."""
import os
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_dx_rows_close, assert_loss_close, from_dev, it, lt, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _run_ranks(W, fn):
    """fn(rank) on W threads (one stream each); re-raises the first failure."""
    out, err = [None] * W, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r)
                s.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            err.append((r, e))

    # daemon threads: a rank stuck in a transport barrier (a protocol bug) cannot keep the process alive
    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "a rank did not finish (loopback transport deadlock?)"
    assert not err, err
    return out


def _loopback(monkeypatch):
    monkeypatch.setenv("F2C_LOOPBACK", "1")
    return os.urandom(128)


@pytest.mark.parametrize("W,C,d,K,dt", [(2, 1000, 128, 1, synth.BF16), (3, 1001, 256, 1, synth.BF16),
                                        (4, 2049, 512, 1, synth.BF16), (3, 700, 128, 2, synth.BF16),
                                        (2, 900, 256, 1, synth.F32)])
def test_loopback_world_steps(dcp, monkeypatch, W, C, d, K, dt):
    uid = _loopback(monkeypatch)
    cfg = synth.scaled(synth.CONFIGS["c1"], name="lb", d=d, C=C, M_loc=24, n_id=2 * C, prefill=0, dtype=dt)
    M, N_loc = cfg.M_loc, cfg.N_loc()
    nblk = cfg.prefill_blocks(W) + 2          # wrapped ring; blocks straddle shard boundaries
    steps = 3
    tdt = torch.bfloat16 if dt == synth.BF16 else torch.float32

    def blk(b, r):
        g, y = synth.prefill_block(cfg, b, r, W)
        if K > 1:
            g = np.stack([g] + [synth.unit_rows(cfg.seed + 7 * k, synth.S_PRE, b, r * M, M, d, dt) for k in range(1, K)],
                         axis=1)
        return g, y

    def step_block(t, r):
        st = synth.step_inputs(cfg, t, r, W)
        g = st.g
        if K > 1:
            g = np.stack([g] + [synth.unit_rows(cfg.seed + 11 * k, synth.S_IDX, t, r * M, M, d, dt) for k in range(1, K)],
                         axis=1)
        return st, g

    def rank_fn(r):
        head = dcp.DCPHead(C, d, dt, W, r, n_local_max=N_loc, m_local_max=M, nccl_uid=uid, K=K)
        for b in range(nblk):
            g, y = blk(b, r)
            head.enqueue(to_dev(g, dt), lt(y))
        res = []
        for t in range(steps):
            st, g = step_block(t, r)
            head.enqueue(to_dev(g, dt), lt(st.gy))
            loss, dx = head.loss_fwd_bwd(to_dev(st.x, dt), lt(st.y), it(st.pairing), cfg.s, cfg.m)
            torch.cuda.current_stream().synchronize()
            res.append((float(loss.item()), from_dev(dx)))
        head.check()
        feats, labs, E = head.get_state()
        head.close()
        return res, feats, labs, E

    out = _run_ranks(W, rank_fn)
    pool = oracle.Pool(C, d, dt, K=K)
    for b in range(nblk):
        parts = [blk(b, r) for r in range(W)]
        pool.enqueue(np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))
    for t in range(steps):
        parts = [step_block(t, r) for r in range(W)]
        pool.enqueue(np.concatenate([p[1] for p in parts]), np.concatenate([p[0].gy for p in parts]))
        X = np.concatenate([p[0].x for p in parts])
        Y = np.concatenate([p[0].y for p in parts])
        PR = np.concatenate([p[0].pairing for p in parts])
        ref = pool.loss(X, Y, PR, cfg.s, cfg.m)
        losses = [out[r][0][t][0] for r in range(W)]
        assert all(v == losses[0] for v in losses), losses      # identical on every rank
        assert_loss_close(losses[0], ref.L)
        gdx = np.concatenate([out[r][0][t][1] for r in range(W)])
        assert_dx_close(gdx, ref.dx)
        assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot < 0)[0], what="dx out-of-pool")
    feats = np.concatenate([out[r][1] for r in range(W)])
    labs = np.concatenate([out[r][2] for r in range(W)])
    assert all(out[r][3] == int(pool.E[0]) for r in range(W))
    np.testing.assert_array_equal(labs, pool.lab)
    np.testing.assert_array_equal(feats[: pool.C_occ], pool.T[: pool.C_occ])


@pytest.mark.parametrize("variant", ["refresh", "excl", "max_hinge", "sum_hinge"])
def test_loopback_world_variants(dcp, monkeypatch, variant):
    """NEXT-3 variants across real per-rank handles: the refresh-in-place enqueue (block all-gather,
    residency MAX all-reduce), stale-duplicate lists after C2, hinge / max partials through C3."""
    uid = _loopback(monkeypatch)
    W, C, d, m_loc, n_loc = 3, 650, 128, 20, 24
    rng = np.random.default_rng(90)
    blocks = []
    for b in range(40):
        G = synth.unit_rows(91, synth.S_PRE, b, 0, W * m_loc, d)
        y = (rng.choice(220, size=W * m_loc, replace=False) if variant == "refresh" else
             rng.integers(0, 220, W * m_loc)).astype(np.int64)
        blocks.append((G, y))
    X = synth.unit_rows(92, synth.S_INST, 0, 0, W * n_loc, d)
    Y = rng.integers(0, 260, W * n_loc).astype(np.int64)
    kw = {}
    if variant == "excl":
        kw = dict(excl_dup=True)
    if variant == "max_hinge":
        kw = dict(phi_mode=oracle.PHI_MAX, hinge=True)
    if variant == "sum_hinge":
        kw = dict(phi_mode=oracle.PHI_SUM, hinge=True, lam=0.5)

    def rank_fn(r):
        head = dcp.DCPHead(C, d, dcp.BF16, W, r, n_local_max=n_loc, m_local_max=m_loc, nccl_uid=uid)
        head.set_enqueue_mode(variant == "refresh")
        head.set_dup_mode(variant == "excl")
        if "phi_mode" in kw:
            head.set_lcos(kw["phi_mode"], kw.get("hinge", False), kw.get("lam", 1.0))
        for G, y in blocks:
            head.enqueue(to_dev(G[r * m_loc:(r + 1) * m_loc], synth.BF16), lt(y[r * m_loc:(r + 1) * m_loc]))
        loss, dx = head.loss_fwd_bwd(to_dev(X[r * n_loc:(r + 1) * n_loc], synth.BF16),
                                     lt(Y[r * n_loc:(r + 1) * n_loc]), None, 64.0, 0.35)
        torch.cuda.current_stream().synchronize()
        head.check()
        feats, labs, E = head.get_state()
        head.close()
        return float(loss.item()), from_dev(dx), labs, E

    out = _run_ranks(W, rank_fn)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, y in blocks:
        pool.enqueue(G, y, refresh=(variant == "refresh"))
    ref = pool.loss(X, Y, None, 64.0, 0.35, **kw)
    assert ref.N_pos > 0 and ref.N_neg > 0
    losses = [o[0] for o in out]
    assert all(v == losses[0] for v in losses)
    assert_loss_close(losses[0], ref.L)
    assert_dx_close(np.concatenate([o[1] for o in out]), ref.dx)
    np.testing.assert_array_equal(np.concatenate([o[2] for o in out]), pool.lab)
    assert all(o[3] == int(pool.E[0]) for o in out)


@pytest.mark.slow
def test_c3_w8_loopback_full_size_sampled_rows(dcp, monkeypatch):
    """BJ:10 at W = 8 through the real per-rank code path: eight handles of 524,288 slots each (global
    batch 8192, global enqueue block 4096, the pool prefilled through C5), one step with pairing;
    sampled rows of ranks 0, 3 and 7 against the single-pool oracle (D16), properties on all rows."""
    from test_gpu_fullsize import _check
    uid = _loopback(monkeypatch)
    cfg, W = synth.CONFIGS["c3"], 8
    M = cfg.M_loc
    nblk = cfg.prefill_blocks(W)
    sts = [synth.step_inputs(cfg, 0, r, W) for r in range(W)]

    def rank_fn(r):
        head = dcp.DCPHead(cfg.C, cfg.d, dcp.BF16, W, r, n_local_max=cfg.N_loc(), m_local_max=M, nccl_uid=uid)
        for b in range(nblk):
            g, y = synth.prefill_block(cfg, b, r, W)
            head.enqueue(to_dev(g, synth.BF16), lt(y))
        st = sts[r]
        head.enqueue(to_dev(st.g, synth.BF16), lt(st.gy))
        loss, dx = head.loss_fwd_bwd(to_dev(st.x, synth.BF16), lt(st.y), it(st.pairing), cfg.s, cfg.m)
        torch.cuda.current_stream().synchronize()
        head.check()
        rs = head.row_stats(cfg.N_loc() * W)
        out = (loss, from_dev(dx), rs)
        head.close()
        return out

    out = _run_ranks(W, rank_fn)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.BF16)
    for b in range(nblk):
        parts = [synth.prefill_block(cfg, b, r, W) for r in range(W)]
        pool.enqueue(np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))
    pool.enqueue(np.concatenate([s.g for s in sts]), np.concatenate([s.gy for s in sts]))
    x = np.concatenate([s.x for s in sts])
    y = np.concatenate([s.y for s in sts])
    pr = np.concatenate([s.pairing for s in sts])
    rng = np.random.default_rng(3)
    rows = np.sort(np.concatenate([r * 2 * M + rng.choice(M, 1, replace=False) for r in (0, 3, 7)] +
                                  [r * 2 * M + M + rng.choice(M, 1, replace=False) for r in (0, 3, 7)]))
    ref = pool.loss_rows(x, y, pr, cfg.s, cfg.m, rows)
    losses = [float(o[0].item()) for o in out]
    assert all(v == losses[0] for v in losses)
    gdx = np.concatenate([o[1] for o in out])
    _check(cfg, out[0][0], gdx, out[0][2], ref, rows)
    assert out[0][2]["N_pos"] >= cfg.M_glob(W)
