"""The shared seeded generator (synth/): pinned to the published splitmix64
reference output, exact [-1, 1) fp32 draws, determinism, range generation
consistency, and the Chinchilla fragment shapes of SURVEY.md §8(d)."""
import numpy as np

import synth


def test_splitmix64_reference_value():
    # splitmix64 with state 0: first output 0xE220A8397B1DCDAF (Vigna's reference)
    assert synth.H(0) == 0xE220A8397B1DCDAF


def test_uniform_draws_exact_and_in_range():
    u = synth.host_U(synth.key(1, 0, 255, 0), 0, 100000)
    assert u.min() >= -1.0 and u.max() < 1.0
    assert np.all(np.mod(u.astype(np.float64) * 2 ** 23, 1.0) == 0.0)  # k * 2^-23 exactly
    assert abs(float(u.mean())) < 0.01


def test_ranges_are_consistent_and_deterministic():
    segs = synth.fragment_segments(64, [0, 3], with_embed=True, vocab=100)
    n = synth.segments_numel(segs)
    full = synth.host_init(segs, 2)
    part = synth.host_init(segs, 2, 1000, 5000)
    assert np.array_equal(full[1000:5000], part)
    w = synth.host_apply_window(full.copy(), segs, 2, 1, 3)
    wp = synth.host_apply_window(full[1000:5000].copy(), segs, 2, 1, 3, i0=1000)
    assert np.array_equal(w[1000:5000], wp)
    assert not np.array_equal(w, synth.host_apply_window(full.copy(), segs, 2, 0, 3))  # private part differs
    assert n == 2 * synth.layer_numel(64) + 100 * 64 + 64


def test_chinchilla_fragment_sizes():
    # 35M |p|=2 -> 6,293,760 (last 22,678,272); 1B |p|=3 -> 151,007,616
    # (last 216,545,664); 4B |p|=3 -> 339,757,440 (last 438,064,512)
    assert synth.segments_numel(synth.fragment_segments(512, [0, 3], False)) == 6293760
    assert synth.segments_numel(synth.fragment_segments(512, [2, 5], True)) == 22678272
    assert synth.segments_numel(synth.fragment_segments(2048, [0, 8, 16], False)) == 151007616
    assert synth.segments_numel(synth.fragment_segments(2048, [7, 15, 23], True)) == 216545664
    assert synth.segments_numel(synth.fragment_segments(3072, [0, 12, 24], False)) == 339757440
    assert synth.segments_numel(synth.fragment_segments(3072, [11, 23, 35], True)) == 438064512


def test_embedding_rows_masked_and_outliers_present():
    d = 256
    segs = synth.fragment_segments(d, [], with_embed=True, vocab=512)
    z = np.zeros(synth.segments_numel(segs), np.float32)
    D = -synth.host_apply_window(z.copy(), segs, 0, 0, 1)
    rows = D[: 512 * d].reshape(512, d)
    zero_rows = (rows == 0).all(axis=1).mean()
    assert 0.35 < zero_rows < 0.65  # "unseen tokens" rows
    big = np.abs(D) > 2.0 ** -9 * 1.5
    assert big.any()  # 2^5 outliers
