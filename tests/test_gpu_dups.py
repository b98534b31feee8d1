"""NEXT-3: the "exclude stale self-duplicates" variant behind
f2c_dcp_set_dup_mode on the GPU path vs the fp64 oracle (orc_loss_v flags bit 1).

Pure Eq. 7 (D7) lets one identity hold several slots.  By default (D8) an in-pool row's older
slots of its own label stay in Eq. 9's denominator; with the variant they are dropped from
that row's softmax.  The pools here draw labels from a small range so that duplicates are
common, and some batch rows are copies of a STALE duplicate's feature (cos = 1 to a slot
that is not the target): there the two readings give clearly different losses, so the test
also checks that the flag changes the result the way the oracle says."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_dx_rows_close, assert_loss_close, from_dev, lt, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _setup(dcp, W, K, C, d, n_loc, m_loc, n_lab, seed, n_blocks=None):
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=n_loc,
                       m_local_max=m_loc, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    nb = n_blocks if n_blocks is not None else C // (m_loc * W) + 2
    for b in range(nb):
        G = synth.unit_rows(seed, synth.S_PRE, b, 0, m_loc * W * K, d)
        if K > 1:
            G = G.reshape(m_loc * W, K, d)
        y = synth.uniform_labels(seed, synth.S_PRE_LAB, b, 0, m_loc * W, n_lab)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    N = W * n_loc
    rng = np.random.default_rng(seed)
    X = synth.unit_rows(seed + 1, synth.S_INST, 0, 0, N, d)
    occ = pool.C_occ
    lab = pool.lab[:occ]
    # in-pool rows: labels of the pool; every 4th row copies the feature of a stale duplicate
    y = lab[rng.integers(0, occ, N)].copy()
    y[1::5] = 10**9 + np.arange(len(y[1::5]))                # out-of-pool rows
    seqs = np.arange(occ)
    E = int(pool.E[0])
    seq_of = seqs + C * ((E - 1 - seqs) // C)
    newest = {}
    for c in range(occ):
        L = int(lab[c])
        if L not in newest or seq_of[c] > seq_of[newest[L]]:
            newest[L] = c
    stale = np.array([c for c in range(occ) if newest[int(lab[c])] != c])
    assert len(stale) > 0
    Tb = oracle.bf16_to_f64(pool.T).reshape(C, K, d).mean(axis=1)
    for i in range(0, N, 4):
        c = int(stale[rng.integers(0, len(stale))])
        y[i] = lab[c]
        v = Tb[c] + 0.05 * rng.standard_normal(d) / np.sqrt(d)
        X[i] = oracle.f64_to_bf16(v / np.linalg.norm(v))
    return head, pool, X, y


@pytest.mark.parametrize("W,K,C,d,n_loc,m_loc,n_lab", [
    (1, 1, 1000, 128, 96, 40, 300),     # C not a multiple of 128, many duplicates
    (1, 1, 700, 256, 200, 64, 120),     # several stale slots per label, same tile as the target
    (1, 2, 900, 128, 80, 50, 250),      # K = 2 pool (NEXT-1)
    (2, 1, 1100, 128, 64, 30, 350),     # emulated world: stale slots on the other shard
    (3, 1, 1000, 256, 48, 20, 200),
])
def test_exclude_stale_duplicates_parity(dcp, W, K, C, d, n_loc, m_loc, n_lab):
    head, pool, X, y = _setup(dcp, W, K, C, d, n_loc, m_loc, n_lab, seed=300 + C + W + K)
    xd, yd = to_dev(X, synth.BF16), lt(y)
    L0, dx0 = head.loss_fwd_bwd(xd, yd, None, 64.0, 0.35)
    L0, dx0 = float(L0.item()), from_dev(dx0)
    head.set_dup_mode(True)
    L1, dx1 = head.loss_fwd_bwd(xd, yd, None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    L1, dx1 = float(L1.item()), from_dev(dx1)
    ref0 = pool.loss(X, y, None, 64.0, 0.35)
    ref1 = pool.loss(X, y, None, 64.0, 0.35, excl_dup=True)
    # the variant matters on these inputs (stale copies dominate those rows' softmax)
    assert abs(ref1.L - ref0.L) > 0.05 * abs(ref0.L)
    assert_loss_close(L0, ref0.L, what="loss (D8)")
    assert_loss_close(L1, ref1.L, what="loss (exclude stale)")
    assert_dx_close(dx0, ref0.dx, what="dx (D8)")
    assert_dx_close(dx1, ref1.dx, what="dx (exclude stale)")
    pos = np.where(ref1.tslot >= 0)[0]
    assert_dx_rows_close(dx1, ref1.dx, pos, what="dx in-pool (exclude stale)")
    st = head.row_stats(len(y))
    assert st["N_pos"] == ref1.N_pos and st["N_neg"] == ref1.N_neg
    np.testing.assert_allclose(st["lse"][pos], ref1.lse[pos], rtol=2e-3, atol=2e-3)
    # switching back reproduces the default bit for bit
    head.set_dup_mode(False)
    L2, dx2 = head.loss_fwd_bwd(xd, yd, None, 64.0, 0.35)
    torch.cuda.synchronize()
    assert float(L2.item()) == L0 and np.array_equal(from_dev(dx2), dx0)


def test_exclude_stale_single_label_pool(dcp):
    """Degenerate: every slot carries the same label, so for rows of that label all but the
    newest slot are stale and the softmax runs over the target alone (L_ce = 0 there)."""
    C, d, m_loc = 520, 128, 64
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=64, m_local_max=m_loc)
    pool = oracle.Pool(C, d, oracle.BF16)
    for b in range(10):
        G = synth.unit_rows(17, synth.S_PRE, b, 0, m_loc, d)
        y = np.full(m_loc, 7, np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    X = synth.unit_rows(18, synth.S_INST, 0, 0, 64, d)
    y = np.full(64, 7, np.int64)
    y[::3] = 8                                                # out-of-pool rows
    head.set_dup_mode(True)
    L, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35, excl_dup=True)
    assert_loss_close(float(L.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    st = head.row_stats(len(y))
    pos = ref.tslot >= 0
    np.testing.assert_allclose(st["ell"][pos], 0.0, atol=1e-5)


def test_dup_mode_bad_args(dcp):
    head = dcp.DCPHead(300, 128, dcp.BF16, 1, 0, n_local_max=16, m_local_max=16)
    lib = dcp.load_library()
    assert lib.f2c_dcp_set_dup_mode(head._h, 2) == 1
    assert lib.f2c_dcp_set_dup_mode(None, 1) == 1
