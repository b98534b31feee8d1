"""NEXT-1: K features per slot (the paper's default K = 2) on the
GPU path vs the fp64 oracle's K-feature pool (orc_loss_k; reading R4).  Raw pool state
bit-exact; loss / dx to the BJ:5 tolerances; world 1 and the emulated world 2."""
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


def _feats(seed, b, m, K, d):
    """m identities x K unit features (each feature its own seeded unit row)."""
    return synth.unit_rows(seed, synth.S_PRE, b, 0, m * K, d).reshape(m, K, d)


def _fill(head, pool, C, K, d, m, n_id, seed, W=1):
    for b in range(C // m + 2):   # wraps
        G = _feats(seed, b, m * W, K, d)
        y = synth.uniform_labels(seed, synth.S_PRE_LAB, b, 0, m * W, n_id)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)


def _batch(pool, C, n, d, n_id, seed):
    X = synth.unit_rows(seed, synth.S_INST, 0, 0, n, d)
    y = synth.uniform_labels(seed, synth.S_INST_LAB, 0, 0, n, n_id)
    y[::3] = pool.lab[: pool.C_occ][(np.arange(len(y[::3])) * 7) % pool.C_occ]
    return X, y


@pytest.mark.parametrize("K,C,d,m", [(2, 1000, 128, 64), (2, 777, 256, 100), (3, 513, 512, 50), (8, 400, 512, 40)])
def test_k_enqueue_state_bit_exact(dcp, K, C, d, m):
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=64, m_local_max=m, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    _fill(head, pool, C, K, d, m, 10**6, seed=40 + K)
    feats, labs, E = head.get_state()
    assert feats.shape == (C, K, d) and E == int(pool.E[0])
    np.testing.assert_array_equal(labs, pool.lab)
    np.testing.assert_array_equal(feats, pool.T)
    head.check()


@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("K,C,d", [(2, 1000, 128), (2, 1301, 256), (3, 900, 512), (8, 700, 512)])
def test_k_loss_parity(dcp, W, K, C, d):
    n_loc, m_loc, n_id = 200, 60, 1500
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=n_loc,
                       m_local_max=m_loc, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    _fill(head, pool, C, K, d, m_loc, n_id, seed=50 + K + d, W=W)
    X, y = _batch(pool, C, W * n_loc, d, n_id, seed=60 + d)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert ref.N_pos > 0 and ref.N_neg > 0
    st = head.row_stats(W * n_loc)
    assert st["N_pos"] == ref.N_pos and st["N_neg"] == ref.N_neg and st["C_occ"] == ref.C_occ
    np.testing.assert_array_equal(np.where(st["target_seq"] >= 0, st["target_seq"] % C, -1), ref.tslot)
    assert_loss_close(float(loss.item()), ref.L)
    pos, neg = ref.tslot >= 0, ref.tslot < 0
    # L_cos with the true cosine (R4): per-row phi of the out-of-pool rows
    np.testing.assert_allclose(st["phi"][neg], ref.phi[neg], rtol=1e-2, atol=2e-4)
    np.testing.assert_allclose(st["ell"][pos], ref.ell[pos], rtol=2e-3, atol=2e-3)
    gdx = from_dev(dx)
    assert_dx_close(gdx, ref.dx)
    assert_dx_rows_close(gdx, ref.dx, np.where(pos)[0], what="dx in-pool")
    assert_dx_rows_close(gdx, ref.dx, np.where(neg)[0], what="dx out-of-pool")


def test_k_zero_center_and_duplicate_features(dcp):
    """Slots whose K features cancel (T_bar = 0: contributes 0 to L_cos) and slots
    whose features coincide (T_bar = f: reduces to the K = 1 pool)."""
    C, d, K, m = 300, 128, 2, 50
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=128, m_local_max=m, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    for b in range(6):
        f = synth.unit_rows(70, synth.S_PRE, b, 0, m, d)
        G = np.stack([f, f], axis=1)
        G[::4, 1] = f[::4] ^ np.uint16(0x8000)     # -f: exact zero center
        y = synth.uniform_labels(70, synth.S_PRE_LAB, b, 0, m, 400)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    X, y = _batch(pool, C, 128, d, 400, seed=71)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 30.0, 0.2)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 30.0, 0.2)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    assert_dx_rows_close(from_dev(dx), ref.dx, np.where(ref.tslot < 0)[0], what="dx out-of-pool")


def test_k_set_state_roundtrip(dcp):
    C, d, K, m = 600, 256, 2, 40
    a = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=96, m_local_max=m, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    for b in range(9):                           # partially filled (E = 360 < C)
        G = _feats(80, b, m, K, d)
        y = synth.uniform_labels(80, synth.S_PRE_LAB, b, 0, m, 500)
        a.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    feats, labs, E = a.get_state()
    b_ = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=96, m_local_max=m, K=K)
    b_.set_state(feats, labs, E)
    f2, l2, E2 = b_.get_state()
    np.testing.assert_array_equal(f2, feats)
    np.testing.assert_array_equal(l2, labs)
    assert E2 == E
    X, y = _batch(pool, C, 96, d, 500, seed=81)
    pr = None
    la, dxa = a.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), pr, 64.0, 0.35)
    lb, dxb = b_.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), pr, 64.0, 0.35)
    torch.cuda.synchronize()
    assert float(la.item()) == float(lb.item())
    assert torch.equal(dxa, dxb)
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert_loss_close(float(lb.item()), ref.L)


def test_k_rejects_f32(dcp):
    with pytest.raises(dcp.DCPError):
        dcp.DCPHead(100, 128, dcp.F32, 1, 0, n_local_max=8, m_local_max=8, K=2)
