"""The shard label index (a3): target resolution (D8: the newest occupied
slot with the row's label) by one lookup per row, the index kept by the enqueue kernels (evict the
overwritten slot's label if that slot held its newest copy, insert the new one) and rebuilt from the
labels when its key count could pass half its capacity.  Checked against the oracle's tslot over
many ring wraps with heavy label reuse (duplicates, evicted labels coming back), several index
rebuilds, refresh-in-place enqueues, set_state and emulated worlds."""
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


@pytest.mark.parametrize("W,C,M,n_lab,refresh", [(1, 300, 37, 90, False), (1, 1000, 64, 5000, False),
                                                 (3, 700, 20, 150, False), (1, 500, 40, 300, True),
                                                 (2, 640, 30, 200, True)])
def test_index_targets_over_many_wraps(dcp, W, C, M, n_lab, refresh):
    d, n_loc = 128, 40
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=n_loc, m_local_max=M)
    head.set_enqueue_mode(refresh)
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(C + M + W)
    Mg = M * W
    nblk = 12 * C // Mg + 5                      # ~12 wraps: several index rebuilds per shard
    checked = 0
    for b in range(nblk):
        G = synth.unit_rows(7, synth.S_PRE, b, 0, Mg, d)
        y = (rng.choice(n_lab, size=Mg, replace=False) if refresh else rng.integers(0, n_lab, Mg)).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=refresh)
        if b % 7 == 3 or b == nblk - 1:
            X = synth.unit_rows(8, synth.S_INST, b, 0, n_loc * W, d)
            yq = rng.integers(0, n_lab + 20, n_loc * W).astype(np.int64)   # some labels never enqueued
            loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(yq), None, 30.0, 0.2)
            torch.cuda.synchronize()
            head.check()
            ref = pool.loss(X, yq, None, 30.0, 0.2)
            st = head.row_stats(n_loc * W)
            np.testing.assert_array_equal(np.where(st["target_seq"] >= 0, st["target_seq"] % C, -1), ref.tslot)
            assert st["N_pos"] == ref.N_pos
            assert_loss_close(float(loss.item()), ref.L)
            assert_dx_close(from_dev(dx), ref.dx)
            checked += 1
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0]) and np.array_equal(labs, pool.lab)
    assert checked >= 5


def test_index_rebuilt_by_set_state(dcp):
    """set_state restores an arbitrary pool (duplicates, partial fill): the index is rebuilt from
    the restored labels, so targets after it equal the oracle's on the same state."""
    d, C, M, n_loc = 128, 400, 50, 32
    rng = np.random.default_rng(5)
    src = oracle.Pool(C, d, oracle.BF16)
    for b in range(11):
        src.enqueue(synth.unit_rows(9, synth.S_PRE, b, 0, M, d), rng.integers(0, 120, M).astype(np.int64))
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=n_loc, m_local_max=M)
    for b in range(3):   # some unrelated state first (its index entries must not survive)
        head.enqueue(to_dev(synth.unit_rows(10, synth.S_PRE, b, 0, M, d), synth.BF16),
                     lt(rng.integers(0, 120, M)))
    head.set_state(src.T, src.lab, int(src.E[0]))
    for step in range(4):
        X = synth.unit_rows(11, synth.S_INST, step, 0, n_loc, d)
        yq = rng.integers(0, 130, n_loc).astype(np.int64)
        loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(yq), None, 64.0, 0.35)
        torch.cuda.synchronize()
        head.check()
        ref = src.loss(X, yq, None, 64.0, 0.35)
        st = head.row_stats(n_loc)
        np.testing.assert_array_equal(np.where(st["target_seq"] >= 0, st["target_seq"] % C, -1), ref.tslot)
        assert_loss_close(float(loss.item()), ref.L)
        G = synth.unit_rows(12, synth.S_PRE, step, 0, M, d)
        yb = rng.integers(0, 120, M).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(yb))
        src.enqueue(G, yb)
