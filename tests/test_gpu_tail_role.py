"""dcp_pc_kernel's tail role (csrc/dcp_tail.cuh): a last row group of <= 32
in-pool rows runs transposed on its own single-CTA ranges (S^T = T x^T, O^T = T^T P^T) instead of as
a CTA pair's unit.  Forced on (F2C_TAIL=1) and off (F2C_TAIL=0) at create, over batches built to
hold exactly 128 k + t in-pool rows (t = 1 .. 32), every d, ragged pools, the R1 refinement pass
(s > 68) and an emulated 2-rank world: loss and dx must match the fp64 oracle (BJ:5), and the
schedule must report the role where it was forced."""
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


def _case(C, d, n_pos, n_out, seed, M=400):
    """A pool filled (and wrapped) by random blocks; a batch whose first n_pos rows have labels in
    the pool and whose other rows have labels no slot holds."""
    rng = np.random.default_rng(seed)
    pool = oracle.Pool(C, d, oracle.BF16)
    blocks = []
    for b in range(C // M + 2):
        G = synth.unit_rows(seed, synth.S_PRE, b, 0, M, d)
        y = rng.choice(50 * C, size=M, replace=False).astype(np.int64)
        blocks.append((G, y))
        pool.enqueue(G, y)
    N = n_pos + n_out
    X = synth.unit_rows(seed + 1, synth.S_INST, 0, 0, N, d)
    lab = pool.lab[: pool.C_occ]
    y = np.empty(N, np.int64)
    y[:n_pos] = rng.choice(np.unique(lab), size=n_pos, replace=False)
    y[n_pos:] = 10**9 + np.arange(n_out)
    perm = rng.permutation(N)  # in-pool rows scattered over the batch
    return blocks, X[perm], y[perm]


CASES = [  # (C, d, n_pos, n_out, s, world)
    (3000, 512, 128 + 23, 40, 64.0, 1),
    (9001, 256, 256 + 1, 17, 64.0, 1),
    (5000, 128, 128 + 32, 0, 30.0, 1),
    (2200, 384, 384 + 7, 9, 64.0, 1),
    (7000, 512, 512 + 16, 30, 100.0, 1),   # s > 68: the R1 refinement pass runs the kernel twice
    (6001, 512, 128 + 20, 36, 64.0, 2),    # emulated world: every shard's own tail role
]


@pytest.mark.parametrize("mode", ["1", "0"])
@pytest.mark.parametrize("C,d,n_pos,n_out,s,world", CASES)
def test_tail_role_parity(dcp, monkeypatch, mode, C, d, n_pos, n_out, s, world):
    monkeypatch.setenv("F2C_TAIL", mode)
    blocks, X, y = _case(C, d, n_pos, n_out, seed=700 + C)
    N = len(y)
    head = dcp.DCPHead(C, d, dcp.BF16, world=world, rank=0 if world == 1 else -1, n_local_max=N // world,
                       m_local_max=400 // world)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yb in blocks:
        head.enqueue(to_dev(G, synth.BF16), lt(yb))
        pool.enqueue(G, yb)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, s, 0.35)
    torch.cuda.synchronize()
    head.check()
    S, tail_G = head.schedule()
    if mode == "1":
        assert tail_G > 0, (S, tail_G)
    else:
        assert tail_G == 0, (S, tail_G)
    ref = pool.loss(X, y, None, s, 0.35)
    assert ref.N_pos == n_pos
    assert_loss_close(float(loss.item()), ref.L, what=f"loss (tail role {mode})")
    assert_dx_close(from_dev(dx), ref.dx, what=f"dx (tail role {mode})")
    st = head.row_stats(N)
    np.testing.assert_allclose(st["lse"][ref.tslot >= 0], ref.lse[ref.tslot >= 0], rtol=2e-5, atol=2e-4)
    head.close()


def test_tail_role_more_ranges_than_tiles(dcp, monkeypatch):
    """A pool of 3 tiles and a forced tail role: most tail CTAs get an empty range."""
    monkeypatch.setenv("F2C_TAIL", "1")
    C, d = 300, 256
    blocks, X, y = _case(C, d, 128 + 5, 3, seed=71, M=150)
    head = dcp.DCPHead(C, d, dcp.BF16, n_local_max=len(y), m_local_max=150)
    pool = oracle.Pool(C, d, oracle.BF16)
    for G, yb in blocks:
        head.enqueue(to_dev(G, synth.BF16), lt(yb))
        pool.enqueue(G, yb)
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    assert head.schedule()[1] > 0
    ref = pool.loss(X, y, None, 64.0, 0.35)
    assert_loss_close(float(loss.item()), ref.L)
    assert_dx_close(from_dev(dx), ref.dx)
    head.close()
