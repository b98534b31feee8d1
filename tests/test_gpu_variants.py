"""NEXT-3: the L_cos variants behind f2c_dcp_set_lcos -- phi = mean /
sum / max over the pool, the hinge max(0, cos), the weight lambda -- on the GPU path vs the
fp64 oracle (orc_loss_v), for K = 1 and K = 2, world 1 and the emulated world 2.

Out-of-pool rows are noisy copies of pool features (labels not in the pool), so the hardest
negative is unique by a wide margin and the bf16 GEMM picks the oracle's slot.  For K = 2
the features are arbitrary bf16 rows: the logits GEMM contracts x with the K raw rows of a
slot, so the cosines (and the hinge decision at cos = 0) use the exact mean (reading R5)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import (assert_dx_close, assert_dx_rows_close, assert_loss_close, from_dev, lt,
                     to_dev)

pytestmark = pytest.mark.gpu

MODES = [(oracle.PHI_MEAN, False, 1.0), (oracle.PHI_SUM, False, 1.0), (oracle.PHI_MEAN, False, 0.0),
         (oracle.PHI_MEAN, True, 1.0), (oracle.PHI_SUM, True, 0.5), (oracle.PHI_MAX, False, 1.0),
         (oracle.PHI_MAX, True, 2.0)]


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _setup(dcp, W, K, C, d, n_loc, m_loc, seed):
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=n_loc,
                       m_local_max=m_loc, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    n_id = 3 * C
    for b in range(C // (m_loc * W) + 2):
        G = synth.unit_rows(seed, synth.S_PRE, b, 0, m_loc * W * K, d)
        if K > 1:  # arbitrary bf16 features, K per slot (NEXT-1: exact-mean logits)
            G = G.reshape(m_loc * W, K, d)
        y = synth.uniform_labels(seed, synth.S_PRE_LAB, b, 0, m_loc * W, n_id)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    N = W * n_loc
    X = synth.unit_rows(seed + 1, synth.S_INST, 0, 0, N, d)
    y = synth.uniform_labels(seed + 1, synth.S_INST_LAB, 0, 0, N, n_id)
    occ = pool.C_occ
    rng = np.random.default_rng(seed)
    y[::2] = pool.lab[:occ][rng.integers(0, occ, len(y[::2]))]   # in-pool half
    neg = np.where(~np.isin(y, pool.lab[:occ]))[0]
    Tb = oracle.bf16_to_f64(pool.T).reshape(C, K, d).mean(axis=1)
    src = rng.integers(0, occ, len(neg))
    v = Tb[src] + 0.25 * rng.standard_normal((len(neg), d)) / np.sqrt(d)
    X[neg] = oracle.f64_to_bf16(v / np.linalg.norm(v, axis=1, keepdims=True))
    return head, pool, X, y


@pytest.mark.parametrize("mode,hinge,lam", MODES)
@pytest.mark.parametrize("W,K", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_lcos_variant_parity(dcp, mode, hinge, lam, W, K):
    C, d, n_loc, m_loc = 900, 256, 160, 50
    head, pool, X, y = _setup(dcp, W, K, C, d, n_loc, m_loc, seed=90 + 7 * K + W)
    head.set_lcos(mode, hinge, lam)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35, phi_mode=mode, hinge=hinge, lam=lam)
    assert ref.N_neg > 0 and ref.N_pos > 0
    st = head.row_stats(len(y))
    assert st["N_pos"] == ref.N_pos and st["N_neg"] == ref.N_neg
    neg, pos = ref.tslot < 0, ref.tslot >= 0
    np.testing.assert_allclose(st["phi"][neg], ref.phi[neg], rtol=1e-2,
                               atol=2e-3 * max(1.0, np.abs(ref.phi[neg]).max()))
    assert_loss_close(float(loss.item()), ref.L)
    gdx = from_dev(dx)
    assert_dx_close(gdx, ref.dx)
    assert_dx_rows_close(gdx, ref.dx, np.where(pos)[0], what="dx in-pool")
    if lam != 0.0:
        assert_dx_rows_close(gdx, ref.dx, np.where(neg)[0], what="dx out-of-pool")
    else:
        assert np.all(gdx[neg] == 0.0)


def test_lcos_variant_switch_back_and_bad_args(dcp):
    """The variant is a handle setting: switching back to the default reproduces the default
    result bit for bit; out-of-range values are rejected (F2C_EINVAL)."""
    head, pool, X, y = _setup(dcp, 1, 1, 600, 128, 96, 40, seed=120)
    a, dxa = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    a, dxa = float(a.item()), dxa.clone()
    head.set_lcos(oracle.PHI_MAX, True, 3.0)
    head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    head.set_lcos()
    b, dxb = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    assert float(b.item()) == a and torch.equal(dxa, dxb)
    for args in ((3, 0, 1.0), (0, 2, 1.0), (0, 0, float("nan"))):
        with pytest.raises(dcp.DCPError) as e:
            head.set_lcos(*args)
        assert e.value.code == 1
