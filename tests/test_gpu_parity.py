"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same
seeded inputs.  Enqueue state and EMA bit-exact; loss
relative error <= 2e-3; max|dx err| <= 1e-2 max|dx| (BJ:5), also applied to the
in-pool and out-of-pool rows separately and to L_ce / L_cos separately."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import (assert_dx_close, assert_dx_rows_close, assert_loss_close, from_dev, it, lt,
                     to_dev)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _head(dcp, C, d, n_max, m_max, dtype=synth.BF16):
    return dcp.DCPHead(C, d, dtype, 1, 0, n_local_max=n_max, m_local_max=m_max)


def _enqueue_both(head, pool, G, y, dtype=synth.BF16):
    head.enqueue(to_dev(G, dtype), lt(y))
    pool.enqueue(G, y)


def _compare_state(head, pool):
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0])
    np.testing.assert_array_equal(labs, pool.lab)
    occ = pool.C_occ
    np.testing.assert_array_equal(feats[:occ], pool.T[:occ])  # bit-exact bytes


# ----------------------------------------------------------------------------- a1 enqueue
@pytest.mark.parametrize("C,M", [(1000, 64), (777, 100), (4096, 512), (130, 130)])
def test_enqueue_bit_exact_with_wrap(dcp, C, M):
    d = 128
    head = _head(dcp, C, d, 64, M)
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(C + M)
    for b in range(2 * C // M + 3):  # fill, then wrap several times (M need not divide C)
        m = int(rng.integers(1, M + 1))
        G = synth.unit_rows(1, synth.S_PRE, b, 0, m, d)
        _enqueue_both(head, pool, G, rng.integers(0, 10**9, m))
        if b % 5 == 0:
            _compare_state(head, pool)
    _compare_state(head, pool)
    head.check()


def test_enqueue_rejects_bad_args(dcp):
    head = _head(dcp, 100, 128, 64, 64)
    with pytest.raises(dcp.DCPError) as e:
        head.enqueue(to_dev(synth.unit_rows(1, 1, 0, 0, 65, 128), synth.BF16), lt(np.arange(65)))
    assert e.value.code == 2
    head.enqueue(to_dev(synth.unit_rows(1, 1, 0, 0, 4, 128), synth.BF16), lt([1, 2, -5, 3]))
    with pytest.raises(dcp.DCPError) as e:
        head.check()
    assert e.value.code == 7


def test_latched_error_reported_by_next_call(dcp):
    """include/f2c_dcp.h: a device-latched error reaches the host through the handle's mapped
    error word; every later enqueue / loss call returns it without launching anything (no
    synchronisation inside the call) until f2c_dcp_check() reports and clears it."""
    d = 128
    head = _head(dcp, 100, d, 8, 8)
    G = to_dev(synth.unit_rows(1, 1, 0, 0, 4, d), synth.BF16)
    head.enqueue(G, lt([1, 2, -5, 3]))           # negative label: latched on the device
    torch.cuda.synchronize()                      # (the latching kernel has finished)
    with pytest.raises(dcp.DCPError) as e:
        head.enqueue(G, lt([1, 2, 4, 3]))
    assert e.value.code == 7 and "negative label" in str(e.value)
    X = to_dev(synth.unit_rows(1, 2, 0, 0, 4, d), synth.BF16)
    with pytest.raises(dcp.DCPError) as e:        # sticky until check()
        head.loss_fwd_bwd(X, lt([1, 2, 4, 3]), None, 64.0, 0.35)
    assert e.value.code == 7
    with pytest.raises(dcp.DCPError) as e:
        head.check()
    assert e.value.code == 7
    head.enqueue(G, lt([1, 2, 4, 3]))             # cleared: calls work again
    head.loss_fwd_bwd(X, lt([1, 2, 4, 3]), None, 64.0, 0.35)
    head.check()
    # a zero-norm batch row (latched by the loss kernels) is reported the same way
    Z = torch.zeros(4, d, dtype=torch.bfloat16, device="cuda")
    head.loss_fwd_bwd(Z, lt([1, 2, 4, 3]), None, 64.0, 0.35)
    torch.cuda.synchronize()
    with pytest.raises(dcp.DCPError) as e:
        head.loss_fwd_bwd(X, lt([1, 2, 4, 3]), None, 64.0, 0.35)
    assert e.value.code == 7 and "zero-norm" in str(e.value)
    with pytest.raises(dcp.DCPError):
        head.check()
    head.check()


def test_binding_validates_arguments(dcp):
    """dcp.py checks dtype, shape, contiguity and device against the handle before any call."""
    d = 128
    head = _head(dcp, 100, d, 8, 8)
    G = to_dev(synth.unit_rows(1, 1, 0, 0, 4, d), synth.BF16)
    with pytest.raises(dcp.DCPError):
        head.enqueue(G.float(), lt([1, 2, 3, 4]))               # fp32 features to a bf16 handle
    with pytest.raises(dcp.DCPError):
        head.enqueue(G, lt([1, 2, 3]))                          # label count
    with pytest.raises(dcp.DCPError):
        head.enqueue(G[:, :64].contiguous(), lt([1, 2, 3, 4]))  # feature width != d
    head.enqueue(G, lt([1, 2, 3, 4]))
    X = to_dev(synth.unit_rows(1, 2, 0, 0, 4, d), synth.BF16)
    with pytest.raises(dcp.DCPError):
        head.loss_fwd_bwd(X, lt([1, 2, 3]), None, 64.0, 0.35)
    with pytest.raises(dcp.DCPError):
        head.loss_fwd_bwd(X, lt([1, 2, 3, 4]).int(), None, 64.0, 0.35)
    with pytest.raises(dcp.DCPError):
        head.loss_fwd_bwd(X.t().contiguous().t(), lt([1, 2, 3, 4]), None, 64.0, 0.35)
    with pytest.raises(dcp.DCPError):
        head.loss_fwd_bwd(X, lt([1, 2, 3, 4]), None, 64.0, 0.35, dx=torch.empty(4, d, device="cuda"))
    with pytest.raises(dcp.DCPError):
        head.set_state(np.zeros((100, d), np.float32), np.full(100, -1, np.int64), 0)
    l1, _ = head.loss_fwd_bwd(X, lt([1, 2, 3, 4]), None, 64.0, 0.35)
    l2, _ = head.loss_fwd_bwd(X, lt([1, 2, 3, 9]), None, 64.0, 0.35)
    torch.cuda.synchronize()
    assert l1.data_ptr() != l2.data_ptr()                       # a fresh loss scalar per call
    head.check()


# ----------------------------------------------------------------------------- a10 EMA
@pytest.mark.parametrize("n", [1, 7, 4096 + 3, 1_000_003])
@pytest.mark.parametrize("m", [0.0, 0.999, 1.0, 0.37])
def test_ema_bit_exact(dcp, n, m):
    p = synth.f32_normal(3, synth.S_EMA_P, n, 0.05)
    g = synth.f32_normal(3, synth.S_EMA_G, n, 0.05)
    ref = oracle.ema(p, g, m)
    gd = torch.from_numpy(g.copy()).cuda()
    dcp.gnet_ema(torch.from_numpy(p).cuda(), gd, m)
    np.testing.assert_array_equal(gd.cpu().numpy(), ref)


# ----------------------------------------------------------------------------- loss
def _run_case(dcp, C, d, blocks, X, y, pairing, s, m, rows_check=True):
    """blocks: list of (G, y) enqueued in order; then one loss call on (X, y)."""
    N = len(y)
    head = _head(dcp, C, d, max(N, 1), max(len(b[1]) for b in blocks))
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yy in blocks:
        _enqueue_both(head, pool, G, yy)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y),
                                 None if pairing is None else it(pairing), s, m)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, pairing, s, m)
    st = head.row_stats(N)
    assert st["N_pos"] == ref.N_pos and st["N_neg"] == ref.N_neg
    np.testing.assert_array_equal(np.where(st["target_seq"] >= 0, st["target_seq"] % C, -1), ref.tslot)
    assert_loss_close(float(loss.item()), ref.L)
    gdx = from_dev(dx)
    assert_dx_close(gdx, ref.dx)
    pos, neg = np.where(ref.tslot >= 0)[0], np.where(ref.tslot < 0)[0]
    if rows_check:
        assert_dx_rows_close(gdx, ref.dx, pos, what="dx in-pool rows")
        assert_dx_rows_close(gdx, ref.dx, neg, what="dx out-of-pool rows")
        if len(pos):
            assert_loss_close(float(np.mean(st["ell"][pos])), ref.L_ce, what="L_ce")
            np.testing.assert_allclose(st["lse"][pos], ref.lse[pos], rtol=1e-3, atol=2e-3)
        if len(neg):
            assert_loss_close(float(np.mean(st["phi"][neg])), ref.L_cos, rtol=5e-3, atol=1e-5,
                              what="L_cos")
    return head, pool, ref


def _random_pool_blocks(C, d, M, nblk, n_id, seed):
    out = []
    for b in range(nblk):
        out.append((synth.unit_rows(seed, synth.S_PRE, b, 0, M, d),
                    synth.uniform_labels(seed, synth.S_PRE_LAB, b, 0, M, n_id)))
    return out


@pytest.mark.parametrize("d", [128, 256, 384, 512])
def test_loss_small_ragged(dcp, d):
    """C not a multiple of the 128-slot tile, N_pos not a multiple of 64, wrap."""
    C, M, n_id = 333, 50, 400
    blocks = _random_pool_blocks(C, d, M, 9, n_id, 5)
    Xi = synth.unit_rows(6, synth.S_INST, 0, 0, 30, d)
    yi = synth.uniform_labels(6, synth.S_INST_LAB, 0, 0, 30, n_id)
    _run_case(dcp, C, d, blocks, Xi, yi, None, 64.0, 0.35)


@pytest.mark.parametrize("s,m", [(64.0, 0.35), (30.0, 0.0), (1.0, 0.0)])
def test_loss_c0_shape_steps(dcp, s, m):
    """c0 (BJ:7) geometry in bf16 (D21): d=128, C=1024 = 16 x 64, 128-row mixed batches,
    fwd+bwd+enqueue for several steps with pairing checked."""
    cfg = synth.scaled(synth.CONFIGS["c0"], dtype=synth.BF16)
    head = _head(dcp, cfg.C, cfg.d, cfg.N_loc(), cfg.M_loc)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.BF16)
    for b in range(cfg.prefill_blocks()):
        G, yy = synth.prefill_block(cfg, b)
        _enqueue_both(head, pool, G, yy)
    for t in range(4):
        stp = synth.step_inputs(cfg, t)
        _enqueue_both(head, pool, stp.g, stp.gy)           # enqueue first (D4)
        loss, dx = head.loss_fwd_bwd(to_dev(stp.x, synth.BF16), lt(stp.y), it(stp.pairing), s, m)
        head.check()
        ref = pool.loss(stp.x, stp.y, stp.pairing, s, m)
        assert ref.N_pos >= cfg.M_loc
        assert_loss_close(float(loss.item()), ref.L)
        gdx = from_dev(dx)
        assert_dx_close(gdx, ref.dx)
        assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot < 0)[0], what="dx out-of-pool")
    _compare_state(head, pool)


@pytest.mark.parametrize("regime", ["literal", "balanced", "peaked"])
def test_loss_noise_regimes(dcp, regime):
    cfg = synth.scaled(synth.CONFIGS["c1"], C=4000, M_loc=256, prefill=16)
    d = cfg.d
    sig = synth.sigma_regime(regime, d)
    blocks = [synth.prefill_block(cfg, b) for b in range(cfg.prefill_blocks())]
    stp = synth.step_inputs(cfg, 0, sigma=sig)
    blocks.append((stp.g, stp.gy))
    _run_case(dcp, cfg.C, d, blocks, stp.x, stp.y, stp.pairing, 64.0, 0.35)


def test_loss_edge_no_inpool_rows(dcp):
    d = 128
    blocks = _random_pool_blocks(200, d, 40, 3, 1000, 7)
    X = synth.unit_rows(8, synth.S_INST, 0, 0, 10, d)
    _run_case(dcp, 200, d, blocks, X, np.arange(5000, 5010), None, 64.0, 0.35)


def test_loss_edge_all_inpool_and_duplicates(dcp):
    """N_neg = 0; duplicate labels in the pool (target = newest, D8) and in the batch."""
    d, C = 256, 150
    rng = np.random.default_rng(2)
    blocks = []
    for b in range(5):
        blocks.append((synth.unit_rows(9, synth.S_PRE, b, 0, 40, d), rng.integers(0, 30, 40)))
    X = synth.unit_rows(9, synth.S_INST, 0, 0, 70, d)
    labs = np.concatenate([blk[1] for blk in blocks])[-C:]
    y = rng.choice(labs, 70)
    _run_case(dcp, C, d, blocks, X, y, None, 64.0, 0.35)


def test_loss_edge_partial_pool_and_unnormalised_rows(dcp):
    d, C = 512, 5000
    blocks = _random_pool_blocks(C, d, 300, 2, 3000, 11)   # 600 of 5000 slots occupied
    X = synth.unit_rows(12, synth.S_INST, 0, 0, 90, d)
    Xf = oracle.bf16_to_f64(X) * np.linspace(0.2, 7.0, 90)[:, None]  # ||x|| != 1
    X = oracle.f64_to_bf16(Xf)
    y = np.concatenate([blocks[1][1][:45], 10**6 + np.arange(45)])
    _run_case(dcp, C, d, blocks, X, y, None, 30.0, 0.2)


def test_pairing_mismatch_is_reported(dcp):
    d, C = 128, 256
    head = _head(dcp, C, d, 8, 8)
    G = synth.unit_rows(1, 1, 0, 0, 8, d)
    head.enqueue(to_dev(G, synth.BF16), lt(np.arange(8)))
    X = synth.unit_rows(1, 2, 0, 0, 8, d)
    head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(np.arange(8)), it(np.arange(8)), 64, 0.35)
    head.check()  # consistent pairing
    head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(np.arange(8)), it(np.roll(np.arange(8), 1)), 64, 0.35)
    with pytest.raises(dcp.DCPError) as e:
        head.check()
    assert e.value.code == 4


def test_set_state_roundtrip(dcp):
    d, C = 128, 300
    head = _head(dcp, C, d, 16, 64)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yy in _random_pool_blocks(C, d, 64, 7, 500, 13):
        _enqueue_both(head, pool, G, yy)
    feats, labs, E = head.get_state()
    h2 = _head(dcp, C, d, 16, 64)
    h2.set_state(feats, labs, E)
    f2, l2, E2 = h2.get_state()
    np.testing.assert_array_equal(f2, feats)
    np.testing.assert_array_equal(l2, labs)
    X = synth.unit_rows(14, 3, 0, 0, 16, d)
    y = np.concatenate([labs[:8], np.arange(10**6, 10**6 + 8)])
    l1, d1 = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64, 0.35)
    l1 = float(l1.item())
    lb, db = h2.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64, 0.35)
    assert l1 == float(lb.item())
    assert torch.equal(d1, db)


def test_determinism(dcp):
    cfg = synth.scaled(synth.CONFIGS["c1"], C=20000, M_loc=512, prefill=40)
    head = _head(dcp, cfg.C, cfg.d, cfg.N_loc(), cfg.M_loc)
    for b in range(cfg.prefill_blocks()):
        G, yy = synth.prefill_block(cfg, b)
        head.enqueue(to_dev(G, synth.BF16), lt(yy))
    stp = synth.step_inputs(cfg, 0)
    head.enqueue(to_dev(stp.g, synth.BF16), lt(stp.gy))   # D4: the step's block first (pairing names it)
    x, y, pr = to_dev(stp.x, synth.BF16), lt(stp.y), it(stp.pairing)
    outs = []
    for _ in range(3):
        l, d = head.loss_fwd_bwd(x, y, pr, 64, 0.35)
        outs.append((l.clone(), d.clone()))
    head.check()
    for l, d in outs[1:]:
        assert torch.equal(l, outs[0][0]) and torch.equal(d, outs[0][1])


@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("s", [64.0, 128.0])
def test_degenerate_all_negative_cosines(dcp, world, s):
    """Every slot points away from every row (cos ~ -0.99): with a single global reference all
    softmax terms would underflow.  The per-row reference (R1) keeps the result exact at
    s = 64; at s = 128 the rows fall below it and the refinement pass (the R1 fallback, run
    for s > 68) re-runs them against their exact maximum (single pool and emulated 2-rank world)."""
    d, C, n = 128, 300, 24
    rng = np.random.default_rng(17)
    u = rng.standard_normal(d)
    u /= np.linalg.norm(u)
    P = -u[None, :] + 0.1 * rng.standard_normal((C, d)) / np.sqrt(d)
    P /= np.linalg.norm(P, axis=1, keepdims=True)
    G = oracle.f64_to_bf16(P)
    labs = rng.integers(0, 50, C)
    X = u[None, :] + 0.1 * rng.standard_normal((n * world, d)) / np.sqrt(d)
    X = oracle.f64_to_bf16(X)
    y = np.concatenate([labs[rng.integers(0, C, n * world - 5)], 1000 + np.arange(5)])
    if world == 1:
        head = _head(dcp, C, d, n, C)
    else:
        head = dcp.DCPHead(C, d, dcp.BF16, world=world, rank=-1, n_local_max=n, m_local_max=C // world)
    pool = oracle.Pool(C, d, oracle.BF16)
    step = C // world * world if world > 1 else C
    head.enqueue(to_dev(G[:step], synth.BF16), lt(labs[:step]))
    pool.enqueue(G[:step], labs[:step])
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, s, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, s, 0.35)
    assert_loss_close(float(loss.item()), ref.L)
    gdx = from_dev(dx)
    assert_dx_close(gdx, ref.dx)
    assert_dx_rows_close(gdx, ref.dx, np.where(ref.tslot >= 0)[0], what="dx in-pool")


@pytest.mark.parametrize("d", [128, 512])
def test_tp64_comparison_kernel_parity(dcp, d, monkeypatch):
    """The first single-CTA design (dcp_tp64_kernel, F2C_KERNEL=tp64) is
    kept as a comparison point: it must meet the same bar."""
    monkeypatch.setenv("F2C_KERNEL", "tp64")
    C, M, n_id = 1500, 100, 2000
    blocks = _random_pool_blocks(C, d, M, 17, n_id, 21)
    X = synth.unit_rows(22, synth.S_INST, 0, 0, 150, d)
    y = synth.uniform_labels(22, synth.S_INST_LAB, 0, 0, 150, n_id)
    y[::2] = blocks[-1][1][: len(y[::2])]        # half the rows in-pool (70+ rows: two 64-row groups)
    _run_case(dcp, C, d, blocks, X, y, None, 64.0, 0.35)


def test_checkpoint_save_load_resume(dcp, tmp_path):
    """Checkpoint / resume: save() after some steps, load() into a fresh handle, continue --
    enqueue state and loss identical to the uninterrupted handle, bit for bit."""
    C, d, M = 900, 128, 60
    a = _head(dcp, C, d, 120, M)
    blocks = _random_pool_blocks(C, d, M, 20, 700, 61)
    for G, y in blocks[:12]:
        a.enqueue(to_dev(G, synth.BF16), lt(y))
    path = str(tmp_path / "pool.npz")
    a.save(path)
    b = _head(dcp, C, d, 120, M)
    b.load(path)
    for G, y in blocks[12:]:
        a.enqueue(to_dev(G, synth.BF16), lt(y))
        b.enqueue(to_dev(G, synth.BF16), lt(y))
    X = synth.unit_rows(62, synth.S_INST, 0, 0, 100, d)
    y = synth.uniform_labels(62, synth.S_INST_LAB, 0, 0, 100, 700)
    y[::3] = blocks[-1][1][: len(y[::3])]
    la, dxa = a.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    la, dxa = float(la.item()), dxa.clone()
    lb, dxb = b.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    assert float(lb.item()) == la and torch.equal(dxa, dxb)
    fa, ya, Ea = a.get_state()
    fb, yb, Eb = b.get_state()
    assert Ea == Eb and np.array_equal(ya, yb) and np.array_equal(fa, fb)
    c = _head(dcp, C + 1, d, 120, M)
    with pytest.raises(dcp.DCPError):
        c.load(path)


@pytest.mark.parametrize("W,C", [(1, 50), (4, 200), (3, 7)])
def test_tiny_pools_and_shards(dcp, W, C):
    """Pools (and shards) smaller than one 128-slot tile, down to 2-3 slots per shard: the TMA
    boxes run past the end of the tensor (zero fill), every shard has a single partial tile."""
    d, m_loc = 128, 1
    while (m_loc + 1) * W <= min(C, 16):
        m_loc += 1
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=24, m_local_max=m_loc)
    pool = oracle.Pool(C, d, oracle.BF16)
    for b in range(2 * C // (m_loc * W) + 2):
        G = synth.unit_rows(71, synth.S_PRE, b, 0, m_loc * W, d)
        y = synth.uniform_labels(71, synth.S_PRE_LAB, b, 0, m_loc * W, 3 * C)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    N = 24 * W
    X = synth.unit_rows(72, synth.S_INST, 0, 0, N, d)
    y = synth.uniform_labels(72, synth.S_INST_LAB, 0, 0, N, 3 * C)
    y[::2] = pool.lab[np.arange(N // 2) % pool.C_occ]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 30.0, 0.2)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 30.0, 0.2)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)


@pytest.mark.parametrize("W", [1, 2])
def test_empty_pool(dcp, W):
    """Before the first enqueue (D9: slots start empty): no row is in-pool, C_occ = 0, so
    L_ce = L_cos = 0 (D10/D11) and dx = 0 -- on the single-rank and the sharded path."""
    C, d = 256, 128
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=16, m_local_max=8)
    pool = oracle.Pool(C, d, oracle.BF16)
    X = synth.unit_rows(81, synth.S_INST, 0, 0, 16 * W, d)
    y = synth.uniform_labels(81, synth.S_INST_LAB, 0, 0, 16 * W, 100)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert ref.L == 0.0 and ref.N_pos == 0 and ref.C_occ == 0
    assert float(loss.item()) == 0.0
    assert np.all(from_dev(dx) == 0.0)


def test_large_batch_multi_unit_schedule(dcp):
    """40,000 rows against a 3,000-slot pool: ~160 row groups, so every cluster runs several
    units in sequence (x_hat reloads, O drains and segment partials per unit), the compaction
    runs on 40 CTAs and the label hash has 131,072 entries."""
    C, d, M, n_id = 3000, 128, 500, 20000
    head = _head(dcp, C, d, 40000, M)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yy in _random_pool_blocks(C, d, M, 8, n_id, 91):
        _enqueue_both(head, pool, G, yy)
    N = 40000
    X = synth.unit_rows(92, synth.S_INST, 0, 0, N, d)
    y = synth.uniform_labels(92, synth.S_INST_LAB, 0, 0, N, n_id)
    y[::3] = pool.lab[np.arange(len(y[::3])) % pool.C_occ]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    rows = np.arange(0, N, 397)
    ref = pool.loss_rows(X, y, None, 64.0, 0.35, rows)
    st = head.row_stats(N)
    assert st["N_pos"] == ref["N_pos"] and st["N_neg"] == ref["N_neg"]
    pos = ref["tslot"] >= 0
    np.testing.assert_allclose(st["lse"][rows][pos], ref["lse"][pos], rtol=1e-3, atol=2e-3)
    gdx = from_dev(dx)
    for sel in (pos, ~pos):
        err = np.abs(gdx[rows][sel] - ref["dx"][sel]).max()
        assert err <= 1e-2 * np.abs(ref["dx"][sel]).max() + 1e-12


@pytest.mark.parametrize("W", [1, 2])
def test_large_scale_refinement_pass(dcp, W):
    """s = 100 on ordinary inputs (mixed in-pool / out-of-pool rows, duplicates, partial pool):
    the refinement pass runs, touches only rows that need it, and the result meets the bar."""
    C, d, M, n_id = 700, 256, 50, 900
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=60, m_local_max=M)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yy in _random_pool_blocks(C, d, M * W, 9, n_id, 95):
        head.enqueue(to_dev(G, synth.BF16), lt(yy))
        pool.enqueue(G, yy)
    X = synth.unit_rows(96, synth.S_INST, 0, 0, 60 * W, d)
    y = synth.uniform_labels(96, synth.S_INST_LAB, 0, 0, 60 * W, n_id)
    y[::2] = pool.lab[np.arange(len(y[::2])) % pool.C_occ]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 100.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 100.0, 0.35)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
