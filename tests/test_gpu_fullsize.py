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


@pytest.mark.slow
def test_c3_full_size_sampled_rows():
    """BJ:10 at W=1 -- the workload bench.py times by default (4,194,304 slots, batch 1024):
    the pool prefilled through the enqueue kernel from the seeded generator, 8 sampled rows
    checked one by one against the oracle, properties on all rows."""
    cfg = synth.CONFIGS["c3"]
    head, loss, gdx, rs, ref, rows = _run(cfg, 8, seed=2)
    _check(cfg, loss, gdx, rs, ref, rows)


@pytest.mark.slow
def test_c3_w8_emulated_full_size_sampled_rows():
    """BJ:10 at W=8 -- the sharded configuration of the scaling run (524,288 slots per rank,
    global batch 8192, global enqueue block 4096) -- through the multi-rank protocol (C1-C5)
    in the emulated world (all eight shards on this device, collectives as device copies):
    sampled rows against the single-pool oracle (D16), properties on all rows."""
    import paper_2105_10375_b200 as dcp
    cfg, W = synth.CONFIGS["c3"], 8
    Mg = cfg.M_glob(W)
    head = dcp.DCPHead(cfg.C, cfg.d, dcp.BF16, world=W, rank=-1, n_local_max=cfg.N_loc(),
                       m_local_max=cfg.M_loc)
    pool = oracle.Pool(cfg.C, cfg.d, oracle.BF16)
    for b in range(cfg.prefill_blocks(W)):
        parts = [synth.prefill_block(cfg, b, r, W) for r in range(W)]
        G = np.concatenate([p[0] for p in parts])
        y = np.concatenate([p[1] for p in parts])
        head.enqueue(to_dev(G, synth.BF16), lt(y))
        pool.enqueue(G, y)
    sts = [synth.step_inputs(cfg, 0, r, W) for r in range(W)]
    g = np.concatenate([s.g for s in sts])
    gy = np.concatenate([s.gy for s in sts])
    head.enqueue(to_dev(g, synth.BF16), lt(gy))
    pool.enqueue(g, gy)
    x = np.concatenate([s.x for s in sts])
    y = np.concatenate([s.y for s in sts])
    pr = np.concatenate([s.pairing for s in sts])
    loss, dx = head.loss_fwd_bwd(to_dev(x, synth.BF16), lt(y), it(pr), cfg.s, cfg.m)
    torch.cuda.synchronize()
    head.check()
    N = len(y)
    rs = head.row_stats(N)
    gdx = from_dev(dx)
    rng = np.random.default_rng(3)
    M = cfg.M_loc
    # rows of ranks 0, 3 and 7: instance rows [r*2M, r*2M+M), identity rows [r*2M+M, (r+1)*2M)
    rows = np.sort(np.concatenate([r * 2 * M + rng.choice(M, 1, replace=False) for r in (0, 3, 7)] +
                                  [r * 2 * M + M + rng.choice(M, 1, replace=False) for r in (0, 3, 7)]))
    ref = pool.loss_rows(x, y, pr, cfg.s, cfg.m, rows)
    _check(cfg, loss, gdx, rs, ref, rows)
    assert Mg == 4096 and rs["N_pos"] >= Mg


@pytest.mark.slow
def test_c4_largest_batch_rank_shape_sampled_rows():
    """BJ:11's largest batch at the 10 % pool, as one rank of W=8 computes it: all 16,384 global
    rows against a 125,000-slot shard (multi-CTA compaction, 129 row groups, one segment per
    unit); 8 sampled rows against the oracle, properties on all rows."""
    base = synth.c4_point(0.10, 16384, world=8)
    cfg = synth.scaled(base, name="c4r_10_16384", C=base.C // 8, M_loc=16384 // 2, n_id=base.n_id // 8)
    head, loss, gdx, rs, ref, rows = _run(cfg, 8, seed=4)
    _check(cfg, loss, gdx, rs, ref, rows)
