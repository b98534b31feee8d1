"""NEXT-3: SPEC's refresh-in-place enqueue (reading
R7) behind f2c_dcp_set_enqueue_mode, on the GPU path vs the oracle (orc_enqueue_refresh).

The pool state (features, labels, E) must be bit-exact after every block; labels come from a
small range so that refreshes, evictions of resident ids (the R7 fixed point) and duplicates
left by earlier pure Eq. 7 enqueues all occur.  The loss after a refresh enqueue is checked
against the oracle, including the pairing check, which then follows each row's actual slot."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_dx_close, assert_loss_close, from_dev, it, lt, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dcp():
    import paper_2105_10375_b200 as m
    m.load_library()
    return m


def _compare(head, pool):
    feats, labs, E = head.get_state()
    assert E == int(pool.E[0])
    np.testing.assert_array_equal(labs, pool.lab)
    occ = pool.C_occ
    np.testing.assert_array_equal(feats[:occ], pool.T[:occ])


def _block(rng, seed, b, m, K, d, n_lab):
    G = synth.unit_rows(seed, synth.S_PRE, b, 0, m * K, d)
    if K > 1:
        G = G.reshape(m, K, d)
    y = rng.choice(n_lab, size=m, replace=False).astype(np.int64)
    return G, y


@pytest.mark.parametrize("W,K,C,d,m_loc,n_lab", [
    (1, 1, 300, 128, 40, 500),     # C not a multiple of the block, frequent residents
    (1, 1, 256, 128, 64, 150),     # most block ids resident; evictions of residents
    (1, 2, 200, 128, 30, 260),     # K = 2 pool (T_bar rebuilt for refreshed slots)
    (2, 1, 301, 128, 25, 400),     # emulated world: residents on the other shard
    (3, 1, 500, 256, 20, 300),
])
def test_refresh_enqueue_state_bit_exact(dcp, W, K, C, d, m_loc, n_lab):
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=16,
                       m_local_max=m_loc, K=K)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    rng = np.random.default_rng(C + W + K)
    seed = 700 + C
    for b in range(4):                        # pure Eq. 7 first: duplicates in the pool
        G, y = _block(rng, seed, b, m_loc * W, K, d, n_lab)
        y[: len(y) // 3] = y[0]               # (pure mode allows repeated labels in a block)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    head.set_enqueue_mode(True)
    for b in range(4, 40):
        G, y = _block(rng, seed, b, m_loc * W, K, d, n_lab)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=True)
        if b % 3 == 0:
            _compare(head, pool)
    _compare(head, pool)
    head.check()
    # back to pure Eq. 7
    head.set_enqueue_mode(False)
    G, y = _block(rng, seed, 99, m_loc * W, K, d, n_lab)
    head.enqueue(to_dev(G, synth.BF16), lt(y))
    pool.enqueue(G, y)
    _compare(head, pool)


@pytest.mark.parametrize("W", [1, 2])
def test_refresh_then_loss_with_pairing(dcp, W):
    """After a refresh enqueue every identity row is in-pool with its own G-Net row as the
    target; the pairing check follows blk_seq; loss and dx match the oracle."""
    C, d, m_loc = 640, 256, 64
    n_lab = 900
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=2 * m_loc,
                       m_local_max=m_loc)
    head.set_enqueue_mode(True)
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(5 + W)
    for b in range(14):
        G, y = _block(rng, 33, b, m_loc * W, 1, d, n_lab)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=True)
    # the batch: per rank M identity rows (noisy copies of the last block) + M instance rows
    Mg = m_loc * W
    Gb = oracle.bf16_to_f64(pool.T[pool.blk_seq % C])
    ids = pool.lab[pool.blk_seq % C]
    X, Y, PR = [], [], []
    for r in range(W):
        sl = slice(r * m_loc, (r + 1) * m_loc)
        v = Gb[sl] + 0.3 * rng.standard_normal((m_loc, d)) / np.sqrt(d)
        inst = rng.standard_normal((m_loc, d))
        X.append(np.concatenate([v, inst]))
        Y.append(np.concatenate([ids[sl], rng.integers(0, n_lab, m_loc)]))
        PR.append(np.concatenate([np.arange(r * m_loc, (r + 1) * m_loc), -np.ones(m_loc)]).astype(np.int32))
    X = oracle.f64_to_bf16(np.concatenate(X))
    Y, PR = np.concatenate(Y), np.concatenate(PR)
    L, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(Y), it(PR), 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, Y, PR, 64.0, 0.35)
    assert ref.N_pos >= Mg
    assert_loss_close(float(L.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    # a pairing that names another block row is caught
    bad = PR.copy()
    bad[0], bad[1] = PR[1], PR[0]
    head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(Y), it(bad), 64.0, 0.35)
    with pytest.raises(dcp.DCPError) as e:
        head.check()
    assert e.value.code == 4


def test_refresh_large_block_and_duplicate_error(dcp):
    """A block larger than the planning CTA (3000 rows > 1024 threads) and a block that repeats
    a label (input error, latched F2C_EDEVICE)."""
    C, d, M = 5000, 128, 3000
    head = dcp.DCPHead(C, d, dcp.BF16, 1, 0, n_local_max=8, m_local_max=M)
    head.set_enqueue_mode(True)
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(11)
    for b in range(4):
        G, y = _block(rng, 44, b, M, 1, d, 6000)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y, refresh=True)
        _compare(head, pool)
    G, y = _block(rng, 44, 9, 8, 1, d, 6000)
    y[3] = y[5]
    head.enqueue(to_dev(G, synth.BF16), lt(y))
    with pytest.raises(dcp.DCPError) as e:
        head.check()
    assert e.value.code == 7
    lib = dcp.load_library()
    assert lib.f2c_dcp_set_enqueue_mode(head._h, 3) == 1
