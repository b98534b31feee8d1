"""Full-size parity (BJ:8 c1, BJ:9 c2) in the launch configuration bench.py times: the
oracle evaluates sampled rows one by one (orc_loss_rows: global N_pos / N_neg / C_occ /
mu, per-row lse, ell, phi, dx); properties that hold at any size are checked on all rows."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import from_dev, it, lt, to_dev

pytestmark = pytest.mark.gpu


def _run(cfg, n_sample, seed=0):
    import paper_2105_10375_b200 as dcp
    head = dcp.DCPHead(cfg.C, cfg.d, dcp.BF16, 1, 0, n_local_max=cfg.N_loc(), m_local_max=cfg.M_loc)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.BF16)
    for b in range(cfg.prefill_blocks()):
        G, y = synth.prefill_block(cfg, b)
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    st = synth.step_inputs(cfg, 0)
    head.enqueue(to_dev(st.g, synth.BF16), lt(st.gy))
    pool.enqueue(st.g, st.gy)
    loss, dx = head.loss_fwd_bwd(to_dev(st.x, synth.BF16), lt(st.y), it(st.pairing), cfg.s, cfg.m)
    torch.cuda.synchronize()
    head.check()
    N = cfg.N_loc()
    rs = head.row_stats(N)
    gdx = from_dev(dx)
    rng = np.random.default_rng(seed)
    rows = np.sort(np.concatenate([rng.choice(cfg.M_loc, n_sample // 2, replace=False),
                                   cfg.M_loc + rng.choice(cfg.M_loc, n_sample // 2, replace=False)]))
    ref = pool.loss_rows(st.x, st.y, st.pairing, cfg.s, cfg.m, rows)
    return head, loss, gdx, rs, ref, rows


def _check(cfg, loss, gdx, rs, ref, rows):
    assert rs["N_pos"] == ref["N_pos"] and rs["N_neg"] == ref["N_neg"] and rs["C_occ"] == ref["C_occ"]
    tsl = np.where(rs["target_seq"][rows] >= 0, rs["target_seq"][rows] % cfg.C, -1)
    np.testing.assert_array_equal(tsl, ref["tslot"])
    pos = ref["tslot"] >= 0
    # per-row loss terms and lse against the oracle
    np.testing.assert_allclose(rs["ell"][rows][pos], ref["ell"][pos], rtol=2e-3, atol=2e-3)
    np.testing.assert_allclose(rs["lse"][rows][pos], ref["lse"][pos], rtol=1e-3, atol=2e-3)
    np.testing.assert_allclose(rs["phi"][rows][~pos], ref["phi"][~pos], rtol=1e-2, atol=2e-5)
    # dx on the sampled rows: the BJ:5 criterion, per row class
    for sel in (pos, ~pos):
        if sel.any():
            err = np.abs(gdx[rows][sel] - ref["dx"][sel]).max()
            assert err <= 1e-2 * np.abs(ref["dx"][sel]).max() + 1e-12
    # the loss is the mean of the per-row terms (any size)
    allpos = rs["target_seq"] >= 0
    L_rows = rs["ell"][allpos].mean() + (rs["phi"][~allpos].mean() if (~allpos).any() else 0.0)
    assert abs(float(loss.item()) - L_rows) <= 1e-4 * abs(L_rows)
    assert np.isfinite(gdx).all()


def test_c1_full_size_sampled_rows():
    cfg = synth.CONFIGS["c1"]
    head, loss, gdx, rs, ref, rows = _run(cfg, 64)
    _check(cfg, loss, gdx, rs, ref, rows)


@pytest.mark.slow
def test_c2_full_size_sampled_rows():
    cfg = synth.CONFIGS["c2"]
    head, loss, gdx, rs, ref, rows = _run(cfg, 16, seed=1)
    _check(cfg, loss, gdx, rs, ref, rows)
