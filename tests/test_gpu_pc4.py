"""The 2-SM pair kernel dcp_pc4_kernel (F2C_KERNEL=pc4: tcgen05 cta_group::2 in 4-CTA clusters,
256-row groups; default variant, d a multiple of 256) against the fp64 oracle: seeded random
configurations (pool sizes with ragged tiles, partial and wrapped pools, batch sizes that
leave 256-row groups mostly padding, emulated worlds, the s > 68 refinement pass), and the
fused-kernel schedule under several cluster counts."""
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


def _case(i):
    rng = np.random.default_rng(5000 + i)
    W = int(rng.choice([1, 1, 2, 3]))
    d = int(rng.choice([256, 512]))
    C = int(rng.integers(max(W, 3), 6000))
    m_loc = int(rng.integers(1, max(2, min(96, C // W) + 1)))
    n_loc = int(rng.integers(1, 700))
    fill = float(rng.choice([0.3, 1.0, 2.5]))
    s = float(rng.choice([1.0, 30.0, 64.0, 100.0]))
    m = float(rng.choice([0.0, 0.35]))
    phi_mode = int(rng.choice([oracle.PHI_MEAN, oracle.PHI_SUM]))
    n_lab = int(rng.integers(max(2, m_loc * W + 1), 4 * C + 10))
    return dict(W=W, d=d, C=C, m_loc=m_loc, n_loc=n_loc, fill=fill, s=s, m=m, phi_mode=phi_mode,
                n_lab=n_lab, seed=6000 + i)


def _run(dcp, c):
    W, d, C, m_loc = c["W"], c["d"], c["C"], c["m_loc"]
    head = dcp.DCPHead(C, d, dcp.BF16, world=W, rank=0 if W == 1 else -1, n_local_max=c["n_loc"],
                       m_local_max=m_loc)
    head.set_lcos(c["phi_mode"], False, 1.0)
    kind, ctas = head.fused_kernel(c["n_loc"] * W)
    assert kind == 2 and ctas > 0 and ctas % 4 == 0, (kind, ctas)  # the cta_group::2 kernel runs
    pool = oracle.Pool(C, d, oracle.BF16)
    rng = np.random.default_rng(c["seed"])
    Mg = m_loc * W
    for b in range(max(1, int(c["fill"] * C / Mg))):
        G = synth.unit_rows(c["seed"], synth.S_PRE, b, 0, Mg, d)
        y = rng.choice(c["n_lab"], size=Mg, replace=False).astype(np.int64)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    N = c["n_loc"] * W
    X = synth.unit_rows(c["seed"] + 1, synth.S_INST, 0, 0, N, d)
    y = rng.integers(0, c["n_lab"], N).astype(np.int64)
    y[::2] = pool.lab[:pool.C_occ][rng.integers(0, pool.C_occ, len(y[::2]))]
    loss, dx = head.loss_fwd_bwd(to_dev(X, synth.BF16), lt(y), None, c["s"], c["m"])
    torch.cuda.synchronize()
    head.check()
    ref = pool.loss(X, y, None, c["s"], c["m"], phi_mode=c["phi_mode"])
    assert_loss_close(float(loss.item()), ref.L, what=f"loss {c}")
    assert_dx_close(from_dev(dx), ref.dx, what=f"dx {c}")


@pytest.mark.parametrize("i", range(int(os.environ.get("F2C_PC4_CASES", "24"))))
def test_pc4_fuzz_parity(dcp, i, monkeypatch):
    monkeypatch.setenv("F2C_KERNEL", "pc4")
    _run(dcp, _case(i))


@pytest.mark.parametrize("clusters", [1, 2, 5, 9])
def test_pc4_cluster_counts(dcp, clusters, monkeypatch):
    # F2C_CLUSTERS counts CTA pairs: 2 * clusters pairs = 4 * clusters SMs = `clusters` four-CTA clusters
    monkeypatch.setenv("F2C_KERNEL", "pc4")
    monkeypatch.setenv("F2C_CLUSTERS", str(2 * clusters))
    _run(dcp, dict(W=1, d=512, C=7000, m_loc=300, n_loc=900, fill=1.3, s=64.0, m=0.35,
                   phi_mode=oracle.PHI_MEAN, n_lab=50000, seed=77))
