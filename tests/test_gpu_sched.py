"""The fused kernel's work schedule (TPSched: units of one 128-row group x one range of pool
tiles, S ranges per group chosen by tp_choose_S, units dealt to clusters round-robin) under
different cluster counts (F2C_CLUSTERS, read at create): one cluster running every unit,
counts that give single and multiple waves, counts that leave clusters idle, and units with
one tile.  Every schedule must give the oracle's loss and dx (the segment partials of a row
are added in a fixed order, so schedules differ only in rounding)."""
import os

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


@pytest.fixture(scope="module")
def case():
    """C = 9000 slots (71 tiles, ragged), d = 256, 400 rows (about 200 in-pool: two row groups)."""
    C, d, M, N = 9000, 256, 500, 400
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(77)
    blocks = []
    for b in range(C // M + 2):  # wraps once
        G = synth.unit_rows(77, synth.S_PRE, b, 0, M, d)
        y = rng.choice(40 * C, size=M, replace=False).astype(np.int64)
        blocks.append((G, y))
        pool.enqueue(G, y)
    X = synth.unit_rows(78, synth.S_INST, 0, 0, N, d)
    y = rng.integers(0, 40 * C, N).astype(np.int64)
    y[::2] = pool.lab[rng.integers(0, C, N // 2)]
    ref = pool.loss(X, y, None, 64.0, 0.35)
    return dict(C=C, d=d, M=M, N=N, blocks=blocks, X=X, y=y, ref=ref)


@pytest.mark.parametrize("clusters", [1, 2, 3, 5, 7, 16, 33, 74])
def test_schedule_cluster_counts(dcp, case, clusters, monkeypatch):
    monkeypatch.setenv("F2C_CLUSTERS", str(clusters))
    head = dcp.DCPHead(case["C"], case["d"], dcp.BF16, world=1, rank=0, n_local_max=case["N"],
                       m_local_max=case["M"])
    kind, ctas = head.fused_kernel(case["N"])
    assert kind == 0 and ctas == 2 * clusters, (kind, ctas)  # dcp_pc_kernel, one CTA pair per cluster
    for G, y in case["blocks"]:
        head.enqueue(to_dev(G, synth.BF16), lt(y))
    loss, dx = head.loss_fwd_bwd(to_dev(case["X"], synth.BF16), lt(case["y"]), None, 64.0, 0.35)
    torch.cuda.synchronize()
    head.check()
    assert_loss_close(float(loss.item()), case["ref"].L, what=f"loss, {clusters} clusters")
    assert_dx_close(from_dev(dx), case["ref"].dx, what=f"dx, {clusters} clusters")
