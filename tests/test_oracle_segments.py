"""Pins for the oracle's many-segment helpers and for error_units (CPU only).

* exact_segment_sums_fp16_array / _fp8_array / exact_segment_sums_bf16 must
  equal the single-array oracles (already pinned against numpy decoding,
  Fraction brute force and closed forms) applied to each slice, for every
  thread split (exact homomorphism).
* within_tolerance_segments must agree with the scalar rational test on
  constructed boundary values (hand-computed tolerances) and on every
  fallback class (specials, g off the 2^-24 grid, values past 2^62 units).
* error_units: hand-computed distances (it had no pin).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

ONE_F16, ONE_BF16 = 0x3C00, 0x3F80


def _random_offsets(rng, n, s):
    off = np.sort(rng.integers(0, n + 1, s + 1))
    off[0] = 0
    return off.astype(np.int64)


def test_error_units_hand_computed():
    es = oracle.exact_sum_fp16(np.array([ONE_F16, ONE_F16], dtype=np.uint16))  # R = 2
    assert es.T == 2 << 24
    assert oracle.error_units(2.0, es) == 0
    assert oracle.error_units(2.0 + 3 * 2.0 ** -24, es) == 3
    assert oracle.error_units(2.0 - 3 * 2.0 ** -24, es) == 3
    assert oracle.error_units(2.0 + 2.0 ** -25, es) == Fraction(1, 2)
    assert oracle.error_units(-2.0, es) == 4 << 24
    # bfloat16: R = 1 + 2^-133 (1.0 plus the smallest subnormal, pattern 0x0001)
    eb = oracle.exact_sum_bf16(np.array([ONE_BF16, 0x0001], dtype=np.uint16))
    assert eb.value == 1 + Fraction(1, 1 << 133)
    assert oracle.error_units(1.0, eb) == Fraction(1, 1 << 109)
    assert oracle.error_units(1.0 + 2.0 ** -20, eb) == 16 - Fraction(1, 1 << 109)
    # fp8 E4M3: 0x38 = 1.0, 0x01 = 2^-9 -> R = 1 + 2^-9; g = 1 is 2^15 units away
    e8 = oracle.exact_sum_fp8(np.array([0x38, 0x01], dtype=np.uint8), oracle.FP8_E4M3)
    assert e8.value == 1 + Fraction(1, 512)
    assert oracle.error_units(1.0, e8) == 1 << 15


def test_segment_arrays_equal_per_slice():
    rng = np.random.default_rng(7)
    n = 200_000
    bits = gen.generate(5, 0, n, gen.WIDE)
    off = _random_offsets(rng, n, 777)
    off[10:20] = off[10]  # a run of empty segments
    ref = [oracle.exact_sum_fp16(bits[off[j]:off[j + 1]]) for j in range(off.size - 1)]
    for threads in (1, 3, 16):
        ss = oracle.exact_segment_sums_fp16_array(bits, off, threads=threads)
        assert len(ss) == len(ref)
        assert all(ss[j] == ref[j] for j in range(len(ref)))
    b8 = gen.generate_fp8(6, 0, n, gen.WIDE, gen.FP8_E5M2)
    for fmt in (oracle.FP8_E4M3, oracle.FP8_E5M2):
        ss = oracle.exact_segment_sums_fp8_array(b8, off, fmt, threads=5)
        for j in range(0, off.size - 1, 7):
            assert ss[j] == oracle.exact_sum_fp8(b8[off[j]:off[j + 1]], fmt)
    bb = gen.generate_bf16(8, 0, 20_000, gen.WIDE)
    offb = _random_offsets(rng, 20_000, 50)
    eb = oracle.exact_segment_sums_bf16(bb, offb)
    assert all(eb[j] == oracle.exact_sum_bf16(bb[offb[j]:offb[j + 1]]) for j in range(50))
    with pytest.raises(ValueError):
        oracle.exact_segment_sums_fp16_array(bits, np.array([0, 5, 3], dtype=np.int64))
    with pytest.raises(ValueError):
        oracle.exact_segment_sums_fp8_array(b8, np.array([0, n + 1], dtype=np.int64), 0)


def test_within_tolerance_segments_boundaries():
    # segment 0: 2^20 ones -> R = 2^20, A = 2^20, tolerance exactly 1.0
    # segment 1: 3 zeros -> R = 0, A = 0: only g = 0 passes
    # segment 2: one NaN -> only NaN passes (fallback path)
    # segment 3: 1.0 and +inf -> only +inf passes
    k = 1 << 20
    bits = np.concatenate([np.full(k, ONE_F16), np.zeros(3), [0x7E00], [ONE_F16, 0x7C00]]
                          ).astype(np.uint16)
    off = np.array([0, k, k + 3, k + 4, k + 6], dtype=np.int64)
    ss = oracle.exact_segment_sums_fp16_array(bits, off)
    cases = [  # (g per segment, expected ok per segment)
        ([2.0 ** 20 + 1, 0.0, float("nan"), float("inf")], [True, True, True, True]),
        ([2.0 ** 20 - 1, -0.0, 1.0, 1.0], [True, True, False, False]),
        ([2.0 ** 20 + 1 + 2.0 ** -24, 2.0 ** -24, float("inf"), float("nan")],
         [False, False, False, False]),
        ([2.0 ** 20 - 1 - 2.0 ** -24, 2.0 ** -30, 0.0, float("-inf")],
         [False, False, False, False]),
        ([2.0 ** 20 + 1 - 2.0 ** -30, float("nan"), float("nan"), float("inf")],  # off-grid g
         [True, False, True, True]),
    ]
    for g, want in cases:
        got = oracle.within_tolerance_segments(np.array(g, dtype=np.float64), ss)
        assert got.tolist() == want, (g, got)
        assert [oracle.within_tolerance(gj, ss[j]) for j, gj in enumerate(g)] == want
    with pytest.raises(ValueError):
        oracle.within_tolerance_segments(np.zeros(3), ss)


def test_within_tolerance_segments_matches_scalar_random():
    rng = np.random.default_rng(11)
    n = 100_000
    for dist in (gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01):
        bits = gen.generate(40 + dist, 0, n, dist)
        off = _random_offsets(rng, n, 400)
        ss = oracle.exact_segment_sums_fp16_array(bits, off)
        exact = np.array([float(ss[j].value) for j in range(len(ss))])
        tol = np.array([float(ss[j].abs_value) * 2.0 ** -20 for j in range(len(ss))])
        # probe just inside / at / outside the tolerance band, on and off the grid
        for scale in (0.0, 0.5, 0.999, 1.0, 1.001, 2.0):
            g = exact + scale * tol * rng.choice([-1.0, 1.0], exact.size)
            g32 = g.astype(np.float32)
            for arr in (g, g32):
                got = oracle.within_tolerance_segments(arr, ss)
                want = [oracle.within_tolerance(float(arr[j]), ss[j]) for j in range(len(ss))]
                assert got.tolist() == want, (dist, scale)


def test_within_tolerance_segments_large_values_fallback():
    # 2^23 copies of 65504 (the largest binary16): T = 2^23 * 65504 * 2^24 > 2^62 units
    # -> the scalar path must decide; g = exact passes, g = 0 fails
    big = np.full(1 << 23, 0x7BFF, dtype=np.uint16)
    ss = oracle.exact_segment_sums_fp16_array(big, np.array([0, big.size], dtype=np.int64))
    assert ss[0].T > 1 << 62
    exact = float(ss[0].value)
    assert oracle.within_tolerance_segments(np.array([exact]), ss).tolist() == [True]
    assert oracle.within_tolerance_segments(np.array([0.0]), ss).tolist() == [False]
