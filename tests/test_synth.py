"""The seeded input generator: determinism, partition
invariance, unit norms, bf16 rounding, label structure (D19, D20)."""
import numpy as np

import oracle
import synth


def test_unit_rows_match_independent_normalise_and_round():
    g = synth.gauss(7, synth.S_INST, 3, 10, 5, 64)
    want = oracle.f64_to_bf16(g / np.linalg.norm(g, axis=1, keepdims=True))
    got = synth.unit_rows(7, synth.S_INST, 3, 10, 5, 64, synth.BF16)
    np.testing.assert_array_equal(got, want)
    got32 = synth.unit_rows(7, synth.S_INST, 3, 10, 5, 64, synth.F32)
    np.testing.assert_array_equal(got32, (g / np.linalg.norm(g, axis=1, keepdims=True)).astype(np.float32))


def test_gaussian_moments_and_determinism():
    a = synth.gauss(1, 2, 3, 0, 400, 128)
    b = synth.gauss(1, 2, 3, 0, 400, 128)
    np.testing.assert_array_equal(a, b)
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1) < 0.01
    # row addressing: rows 100.. generated alone equal the slice
    np.testing.assert_array_equal(synth.gauss(1, 2, 3, 100, 7, 128), a[100:107])


def test_pair_rows_noise_regimes():
    d = 512
    for regime, lo, hi in (("literal", 0.10, 0.20), ("balanced", 0.55, 0.70), ("peaked", 0.94, 0.98)):
        x, g = synth.pair_rows(5, 0, 0, 256, d, synth.sigma_regime(regime, d), synth.BF16)
        xf, gf = oracle.bf16_to_f64(x), oracle.bf16_to_f64(g)
        cos = np.sum(xf * gf, 1) / np.linalg.norm(xf, axis=1) / np.linalg.norm(gf, axis=1)
        assert lo < cos.mean() < hi, (regime, cos.mean())


def test_identity_labels_distinct_and_cover_epoch():
    n_id, M = 1000, 64
    per = n_id // M
    blocks = [synth.identity_labels(9, b, 0, M, M, n_id) for b in range(per)]
    allv = np.concatenate(blocks)
    assert len(set(allv.tolist())) == len(allv)          # no repeats within an epoch
    assert allv.min() >= 0 and allv.max() < n_id
    # rank slices of a block are the block's rows
    full = synth.identity_labels(9, 3, 0, 4 * M, 4 * M, n_id)
    np.testing.assert_array_equal(synth.identity_labels(9, 3, 2 * M, M, 4 * M, n_id), full[2 * M:3 * M])
    # next epoch is reshuffled
    nxt = synth.identity_labels(9, per, 0, M, M, n_id)
    assert not np.array_equal(nxt, blocks[0])


def test_step_inputs_partition_invariant():
    cfg = synth.scaled(synth.CONFIGS["c0"], M_loc=16)
    W = 4
    parts = [synth.step_inputs(cfg, 2, r, W) for r in range(W)]
    whole_ids = synth.identity_labels(cfg.seed, 2, 0, 16 * W, 16 * W, cfg.n_id)
    np.testing.assert_array_equal(np.concatenate([p.gy for p in parts]), whole_ids)
    for r, p in enumerate(parts):
        assert p.x.shape == (32, cfg.d)
        assert (p.pairing[:16] == -1).all() and (p.pairing[16:] == r * 16 + np.arange(16)).all()
        np.testing.assert_array_equal(p.y[16:], p.gy)


def test_uniform_labels_range():
    y = synth.uniform_labels(1, 4, 0, 0, 10000, 37)
    assert y.min() == 0 and y.max() == 36
    assert abs(np.bincount(y).std() / np.bincount(y).mean()) < 0.1
