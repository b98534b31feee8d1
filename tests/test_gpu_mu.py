"""The pool sum mu of the L_cos gradient (reading R3): kept by the enqueue as an exact 64-bit
fixed-point running sum (k_mu_sum), one rounding per slot contribution.

Exactness is checked without the oracle: after many wrapped enqueues (every slot overwritten
several times, in pure Eq. 7 and refresh-in-place order), a second handle restored from the
first one's state (set_state rebuilds mu from scratch in one pass) must give a BIT-identical
loss and dx on a batch of out-of-pool rows -- the rest of the loss path is deterministic, so
any drift or order dependence of the running sum would show.  The oracle comparison of the
same batch (fp64 fresh sum, BJ:5 tolerances) is the parity half."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_loss_close, from_dev, lt, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("W,K,dtype,C,d,m_loc,nblk,refresh", [
    (1, 1, 0, 700, 512, 64, 60, False),     # ~5.5 wraps of a bf16 pool
    (1, 2, 0, 500, 128, 50, 40, True),      # K = 2 with refresh-in-place
    (1, 2, 0, 400, 256, 40, 35, False),     # K = 2: contributions w_c * T_bar_c
    (2, 1, 0, 641, 384, 30, 50, False),     # emulated world: one sum per shard
    (1, 1, 0, 600, 128, 48, 40, True),      # refresh-in-place destinations
])
def test_mu_running_sum_exact(dcp, W, K, dtype, C, d, m_loc, nblk, refresh):
    # (dtype 1, fp32 pools, has no loss path in this build: DESIGN.md D21)
    tdt = synth.BF16 if dtype == 0 else synth.F32
    odt = oracle.BF16 if dtype == 0 else oracle.F32
    rank = 0 if W == 1 else -1
    n_loc = 24
    head = dcp.DCPHead(C, d, dtype, world=W, rank=rank, n_local_max=n_loc, m_local_max=m_loc, K=K)
    head.set_enqueue_mode(refresh)
    pool = oracle.Pool(C, d, odt, K=K)
    rng = np.random.default_rng(C * 7 + d)
    Mg = m_loc * W
    n_lab = 3 * C if refresh else 50 * C
    for b in range(nblk):
        G = synth.unit_rows(900 + C, synth.S_PRE, b, 0, Mg * K, d, dtype=tdt)
        if K > 1:  # arbitrary bf16 features, K per slot (NEXT-1: exact-mean logits)
            G = G.reshape(Mg, K, d)
        y = rng.choice(n_lab, size=Mg, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, tdt), lt(y))
        pool.enqueue(G, y, refresh=refresh)
    # out-of-pool batch (labels above every pool label): the mu path only
    N = n_loc * W
    X = synth.unit_rows(901 + C, synth.S_INST, 0, 0, N, d, dtype=tdt)
    y = (n_lab + np.arange(N)).astype(np.int64)
    loss1, dx1 = head.loss_fwd_bwd(to_dev(X, tdt), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    dx1 = from_dev(dx1)
    # restored copy: mu rebuilt from the restored slots in one pass
    feats, labs, E = head.get_state()
    head2 = dcp.DCPHead(C, d, dtype, world=W, rank=rank, n_local_max=n_loc, m_local_max=m_loc, K=K)
    head2.set_state(feats, labs, E)
    loss2, dx2 = head2.loss_fwd_bwd(to_dev(X, tdt), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head2.check()
    assert float(loss1.item()) == float(loss2.item())
    np.testing.assert_array_equal(dx1.view(np.uint8), from_dev(dx2).view(np.uint8))
    # parity: the oracle's fresh fp64 sum over the pool
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert_loss_close(float(loss1.item()), ref.L, what="loss")
    assert_dx_close(dx1, ref.dx, what="dx")
