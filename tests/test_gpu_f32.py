"""fp32 pools (F2C_F32; BJ:7's c0 is fp32, reading D21): the loss path with tf32 logits -- GEMM 1 in
tcgen05 kind::tf32 over the fp32 rows, x_hat as fp32 in TMEM -- and the P x pool GEMM on the pool's bf16
shadow kept by the enqueue.  Against the fp64 oracle on the same fp32 inputs: enqueue state bit-exact,
loss within 2e-3 and dx within 1e-2 max|dx| (BJ:5), for the c0 steps, the NEXT-3 variants, an emulated
2-rank world and a set_state round trip."""
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


def _compare_state(head, pool):
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0])
    np.testing.assert_array_equal(labs, pool.lab)
    np.testing.assert_array_equal(feats[: pool.C_occ], pool.T[: pool.C_occ])


def test_c0_fp32_steps(dcp):
    """c0 as BASELINE.json states it (BJ:7): d = 128, C = 1024 (16 blocks of 64), N = 128, fp32,
    s = 64, m = 0.35, pool prefilled with 16 enqueues, 20 steps of enqueue + loss."""
    cfg = synth.CONFIGS["c0"]
    assert cfg.dtype == synth.F32
    head = dcp.DCPHead(cfg.C, cfg.d, dcp.F32, 1, 0, n_local_max=cfg.N_loc(), m_local_max=cfg.M_loc)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.F32)
    for b in range(cfg.prefill_blocks()):
        g, y = synth.prefill_block(cfg, b)
        head.enqueue(to_dev(g, synth.F32), lt(y))
        pool.enqueue(g, y)
    for t in range(cfg.steps):
        st = synth.step_inputs(cfg, t)
        head.enqueue(to_dev(st.g, synth.F32), lt(st.gy))
        pool.enqueue(st.g, st.gy)
        loss, dx = head.loss_fwd_bwd(to_dev(st.x, synth.F32), lt(st.y), it(st.pairing), cfg.s, cfg.m)
        torch.cuda.synchronize()
        head.check()
        ref = pool.loss(st.x, st.y, st.pairing, cfg.s, cfg.m)
        assert dx.dtype == torch.float32
        assert_loss_close(float(loss.item()), ref.L)
        gdx = from_dev(dx)
        assert_dx_close(gdx, ref.dx)
        assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot >= 0)[0], what="dx in-pool")
        assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot < 0)[0], what="dx out-of-pool")
        if t % 5 == 0:
            _compare_state(head, pool)
            stt = head.row_stats(cfg.N_loc())
            np.testing.assert_array_equal(np.where(stt["target_seq"] >= 0, stt["target_seq"] % cfg.C, -1), ref.tslot)


@pytest.mark.parametrize("d,C,sigma", [(128, 777, "balanced"), (256, 3000, "peaked"), (256, 300, "literal")])
def test_fp32_noise_regimes(dcp, d, C, sigma):
    cfg = synth.scaled(synth.CONFIGS["c0"], d=d, C=C, M_loc=48, n_id=3 * C)
    sig = synth.sigma_regime(sigma, d)
    head = dcp.DCPHead(C, d, dcp.F32, 1, 0, n_local_max=cfg.N_loc(), m_local_max=cfg.M_loc)
    pool = oracle.Pool(C, d, oracle.F32)
    for b in range(cfg.prefill_blocks() + 3):
        g, y = synth.prefill_block(cfg, b)
        head.enqueue(to_dev(g, synth.F32), lt(y))
        pool.enqueue(g, y)
    st = synth.step_inputs(cfg, 0, sigma=sig)
    head.enqueue(to_dev(st.g, synth.F32), lt(st.gy))
    pool.enqueue(st.g, st.gy)
    loss, dx = head.loss_fwd_bwd(to_dev(st.x, synth.F32), lt(st.y), it(st.pairing), 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(st.x, st.y, st.pairing, 64.0, 0.35)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)


@pytest.mark.parametrize("variant", ["max_hinge", "sum", "excl", "refresh"])
def test_fp32_variants(dcp, variant):
    d, C, m_loc, n = 128, 900, 40, 64
    head = dcp.DCPHead(C, d, dcp.F32, 1, 0, n_local_max=n, m_local_max=m_loc)
    pool = oracle.Pool(C, d, oracle.F32)
    kw = {}
    if variant == "max_hinge":
        head.set_lcos(oracle.PHI_MAX, True, 1.0)
        kw = dict(phi_mode=oracle.PHI_MAX, hinge=True)
    if variant == "sum":
        head.set_lcos(oracle.PHI_SUM, False, 0.5)
        kw = dict(phi_mode=oracle.PHI_SUM, lam=0.5)
    if variant == "excl":
        head.set_dup_mode(True)
        kw = dict(excl_dup=True)
    refresh = variant == "refresh"
    head.set_enqueue_mode(refresh)
    rng = np.random.default_rng(71)
    for b in range(30):
        G = synth.unit_rows(72, synth.S_PRE, b, 0, m_loc, d, synth.F32)
        y = (rng.choice(300, size=m_loc, replace=False) if refresh else rng.integers(0, 300, m_loc)).astype(np.int64)
        head.enqueue(to_dev(G, synth.F32), lt(y))
        pool.enqueue(G, y, refresh=refresh)
    _compare_state(head, pool)
    X = synth.unit_rows(73, synth.S_INST, 0, 0, n, d, synth.F32)
    y = rng.integers(0, 340, n).astype(np.int64)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.F32), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35, **kw)
    assert ref.N_pos > 0 and ref.N_neg > 0
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)


def test_fp32_emulated_world_and_set_state(dcp):
    W, C, d, m_loc, n_loc = 3, 1001, 256, 30, 40
    head = dcp.DCPHead(C, d, dcp.F32, world=W, rank=-1, n_local_max=n_loc, m_local_max=m_loc)
    pool = oracle.Pool(C, d, oracle.F32)
    rng = np.random.default_rng(5)
    for b in range(C // (W * m_loc) + 3):
        G = synth.unit_rows(81, synth.S_PRE, b, 0, W * m_loc, d, synth.F32)
        y = rng.integers(0, 1500, W * m_loc).astype(np.int64)
        head.enqueue(to_dev(G, synth.F32), lt(y))
        pool.enqueue(G, y)
    X = synth.unit_rows(82, synth.S_INST, 0, 0, W * n_loc, d, synth.F32)
    y = rng.integers(0, 1500, W * n_loc).astype(np.int64)
    y[::4] = pool.lab[rng.integers(0, C, len(y[::4]))]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.F32), lt(y), None, 30.0, 0.2)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 30.0, 0.2)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    # set_state into a fresh single-pool fp32 handle rebuilds the bf16 shadow: same loss
    one = dcp.DCPHead(C, d, dcp.F32, 1, 0, n_local_max=W * n_loc, m_local_max=m_loc)
    one.set_state(pool.T, pool.lab, int(pool.E[0]))
    l1, dx1 = one.loss_fwd_bwd(to_dev(X, synth.F32), lt(y), None, 30.0, 0.2)
    torch.cuda.synchronize()
    one.check()
    assert_loss_close(float(l1.item()), ref.L)
    assert_dx_close(from_dev(dx1), ref.dx)


def test_fp32_rejects_wide_features_in_the_loss(dcp):
    head = dcp.DCPHead(500, 384, dcp.F32, 1, 0, n_local_max=8, m_local_max=8)
    head.enqueue(to_dev(synth.unit_rows(1, 1, 0, 0, 8, 384, synth.F32), synth.F32), lt(np.arange(8)))
    with pytest.raises(dcp.DCPError) as e:
        head.loss_fwd_bwd(to_dev(synth.unit_rows(1, 2, 0, 0, 8, 384, synth.F32), synth.F32), lt(np.arange(8)),
                          None, 64.0, 0.35)
    assert e.value.code == 1
    head.check()
