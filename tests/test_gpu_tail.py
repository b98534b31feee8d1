"""The fused kernel's 64-row tail unit (a last row group of at most 64 in-pool rows runs both
GEMMs with M = 64, its rows on TMEM lanes 0-15 of each quadrant) around its boundaries: exactly
N_pos in-pool rows for N_pos in {1, 16, 17, 63, 64, 65, 127, 128, 129, 191, 192, 193}, against
the fp64 oracle, with the stale-duplicate exclusion (NEXT-3) on and off, for the d-block
layouts of d = 256 / 384 / 512 and K = 2."""
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


@pytest.mark.parametrize("n_pos", [1, 16, 17, 63, 64, 65, 127, 128, 129, 191, 192, 193])
@pytest.mark.parametrize("d,K,excl", [(512, 1, False), (384, 1, True), (256, 2, False)])
def test_tail_unit_boundaries(dcp, n_pos, d, K, excl):
    C, M, N = 3000, 250, 240
    head = dcp.DCPHead(C, d, dcp.BF16, world=1, rank=0, n_local_max=N, m_local_max=M, K=K)
    head.set_dup_mode(excl)
    pool = oracle.Pool(C, d, oracle.BF16, K=K)
    rng = np.random.default_rng(n_pos * 7 + d + K)
    for b in range(C // M + 3):  # wraps; small label range: stale duplicates exist
        G = synth.unit_rows(40 + d, synth.S_PRE, b, 0, M * K, d)
        if K > 1:
            G = np.clip(np.rint(oracle.bf16_to_f64(G) * 512), -127, 127) / 512
            G = oracle.f64_to_bf16(G).reshape(M, K, d)
        y = rng.choice(2 * C, size=M, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    X = synth.unit_rows(41 + d, synth.S_INST, 0, 0, N, d)
    y = np.arange(10 * C, 10 * C + N, dtype=np.int64)  # out of pool
    rows = rng.choice(N, size=min(n_pos, N), replace=False)
    y[rows] = pool.lab[rng.integers(0, pool.C_occ, len(rows))]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, 64.0, 0.35, excl_dup=excl)
    assert head.row_stats(N)["N_pos"] == min(n_pos, N)
    assert_loss_close(float(loss.item()), ref.L, what=f"loss n_pos={n_pos}")
    assert_dx_close(from_dev(dx), ref.dx, what=f"dx n_pos={n_pos}")
