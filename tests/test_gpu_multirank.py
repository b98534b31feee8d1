"""Multi-rank path on one GPU: the emulated world (rank = -1) runs every shard's kernels
and the C1-C5 protocol with device copies in place of NCCL.  Results must equal the
single-pool oracle on the rank-ordered concatenated batch and blocks (D16, pin P9)."""
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


@pytest.mark.parametrize("W,C,d", [(2, 1000, 128), (3, 1001, 256), (4, 2048, 512), (8, 4097, 512)])
def test_emulated_world_matches_single_pool(dcp, W, C, d):
    m_loc, n_loc, n_id = 40, 48, 600
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=-1, n_local_max=n_loc, m_local_max=m_loc)
    pool = oracle.Pool(C, d, oracle.BF16)
    nblk = (C // (W * m_loc)) + 2          # wraps; blocks straddle shard boundaries
    for b in range(nblk):
        G = synth.unit_rows(21, synth.S_PRE, b, 0, W * m_loc, d)
        y = synth.uniform_labels(21, synth.S_PRE_LAB, b, 0, W * m_loc, n_id)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    feats, labs, E = head.get_state()
    np.testing.assert_array_equal(labs, pool.lab)
    np.testing.assert_array_equal(feats[: pool.C_occ], pool.T[: pool.C_occ])
    # global batch: per rank, instance rows + rows whose labels are in the last block
    X = synth.unit_rows(22, synth.S_INST, 0, 0, W * n_loc, d)
    y = synth.uniform_labels(22, synth.S_INST_LAB, 0, 0, W * n_loc, n_id)
    last = pool.lab[(int(pool.E[0]) - 1) % C]
    y[::5] = last
    y[1::7] = pool.lab[: pool.C_occ][np.arange(len(y[1::7])) * 13 % pool.C_occ]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35)
    st = head.row_stats(W * n_loc)
    assert st["N_pos"] == ref.N_pos and st["N_neg"] == ref.N_neg
    np.testing.assert_array_equal(np.where(st["target_seq"] >= 0, st["target_seq"] % C, -1), ref.tslot)
    assert_loss_close(float(loss.item()), ref.L)
    gdx = from_dev(dx)
    assert_dx_close(gdx, ref.dx)
    assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot >= 0)[0], what="dx in-pool")
    assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot < 0)[0], what="dx out-of-pool")
    pos = ref.tslot >= 0
    np.testing.assert_allclose(st["lse"][pos], ref.lse[pos], rtol=1e-3, atol=2e-3)


def test_emulated_world_c0_steps_with_pairing(dcp):
    """c0 geometry (bf16, D21) sharded over 4 emulated ranks, several steps with the
    enqueue routed to the owners and pairing checked against the global block."""
    W = 4
    cfg = synth.scaled(synth.CONFIGS["c0"], dtype=synth.BF16, M_loc=16)
    head = dcp.DCPHead(cfg.C, cfg.d, dcp.BF16, world=W, rank=-1, n_local_max=cfg.N_loc(),
                       m_local_max=cfg.M_loc)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.BF16)
    for b in range(cfg.prefill_blocks(W)):
        parts = [synth.prefill_block(cfg, b, r, W) for r in range(W)]
        G = np.concatenate([p[0] for p in parts])
        yy = np.concatenate([p[1] for p in parts])
        head.enqueue(to_dev(G, synth.BF16), lt(yy))
        pool.enqueue(G, yy)
    for t in range(3):
        parts = [synth.step_inputs(cfg, t, r, W) for r in range(W)]
        G = np.concatenate([p.g for p in parts])
        gy = np.concatenate([p.gy for p in parts])
        head.enqueue(to_dev(G, synth.BF16), lt(gy))
        pool.enqueue(G, gy)
        X = np.concatenate([p.x for p in parts])
        y = np.concatenate([p.y for p in parts])
        pr = np.concatenate([p.pairing for p in parts])
        loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), it(pr), cfg.s, cfg.m)
        head.check()
        ref = pool.loss(X, y, pr, cfg.s, cfg.m)
        assert_loss_close(float(loss.item()), ref.L)
        assert_dx_close(from_dev(dx), ref.dx)


def test_nccl_transport_single_rank(dcp, monkeypatch):
    """The NCCL transport of the multi-rank protocol (C1 all-gather, C2 MAX all-reduce,
    C3 all-gather, C4 reduce-scatter, C5 enqueue all-gather) on a real 1-rank NCCL
    communicator (test hook F2C_FORCE_MULTI=1): results must equal the single-pool oracle."""
    monkeypatch.setenv("F2C_FORCE_MULTI", "1")
    C, d, m_loc, n = 700, 256, 50, 40
    head = dcp.DCPHead(C, d, dcp.BF16, world=1, rank=0, n_local_max=n, m_local_max=m_loc)
    monkeypatch.delenv("F2C_FORCE_MULTI")
    pool = oracle.Pool(C, d, oracle.BF16)
    for b in range(16):
        G = synth.unit_rows(31, synth.S_PRE, b, 0, m_loc, d)
        y = synth.uniform_labels(31, synth.S_PRE_LAB, b, 0, m_loc, 300)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    X = synth.unit_rows(32, synth.S_INST, 0, 0, n, d)
    y = synth.uniform_labels(32, synth.S_INST_LAB, 0, 0, n, 300)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    feats, labs, E = head.get_state()
    np.testing.assert_array_equal(labs, pool.lab)


@pytest.mark.parametrize("K,variant", [(1, "refresh"), (1, "excl"), (2, "max_hinge"), (2, "refresh")])
def test_nccl_transport_single_rank_variants(dcp, monkeypatch, K, variant):
    """The NEXT-1 / NEXT-3 variants through the real NCCL transport (1-rank communicator):
    the refresh-in-place enqueue's residency MAX all-reduce, the stale-duplicate lists built
    after C2, the hinge / max partials in C3 -- all against the single-pool oracle."""
    monkeypatch.setenv("F2C_FORCE_MULTI", "1")
    C, d, m_loc, n = 650, 128, 40, 48
    head = dcp.DCPHead(C, d, dcp.BF16, world=1, rank=0, n_local_max=n, m_local_max=m_loc, K=K)
    monkeypatch.delenv("F2C_FORCE_MULTI")
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    if variant == "refresh":
        head.set_enqueue_mode(True)
    if variant == "excl":
        head.set_dup_mode(True)
    if variant == "max_hinge":
        head.set_lcos(oracle.PHI_MAX, True, 1.0)
    rng = np.random.default_rng(40 + K)
    for b in range(24):
        G = synth.unit_rows(41, synth.S_PRE, b, 0, m_loc * K, d)
        if K > 1:  # arbitrary bf16 features, K per slot (NEXT-1: exact-mean logits)
            G = G.reshape(m_loc, K, d)
        y = rng.choice(200, size=m_loc, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=(variant == "refresh"))
    X = synth.unit_rows(42, synth.S_INST, 0, 0, n, d)
    y = rng.integers(0, 260, n).astype(np.int64)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    kw = {}
    if variant == "excl":
        kw = dict(excl_dup=True)
    if variant == "max_hinge":
        kw = dict(phi_mode=oracle.PHI_MAX, hinge=True)
    ref = pool.loss(X, y, None, 64.0, 0.35, **kw)
    assert ref.N_pos > 0 and ref.N_neg > 0
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0])
    np.testing.assert_array_equal(labs, pool.lab)
