"""Pins for oracle.exact_sum_fp16 / round_to_f32 / within_tolerance (CPU only).

Every check here compares the oracle against something other than itself:
numpy's binary16 decoding, Python's Fraction arithmetic, math.fsum
(Shewchuk, correctly rounded), closed forms, and invariants (DESIGN.md
§"Oracle and pins").
"""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

ALL_FINITE = np.array([h for h in range(1 << 16) if ((h >> 10) & 0x1F) != 0x1F], dtype=np.uint16)


def test_all_finite_patterns_decode_like_numpy():
    # Exhaustive: 63 488 finite binary16 patterns; each segment is one element.
    assert ALL_FINITE.size == 63488
    off = np.arange(ALL_FINITE.size + 1, dtype=np.int64)
    res = oracle.exact_segment_sums_fp16(ALL_FINITE, off)
    ref = ALL_FINITE.view(np.float16).astype(np.float64)
    for r, v in zip(res, ref.tolist()):
        assert r.value == Fraction(v)
        assert r.A == abs(r.T)


def test_sum_of_all_finite_patterns_vs_fraction_and_fsum():
    es = oracle.exact_sum_fp16(ALL_FINITE)
    # Every positive pattern has a negative twin: exact sum is 0, sum|x| is twice the positive half.
    assert es.T == 0
    pos = ALL_FINITE[ALL_FINITE < 0x8000].view(np.float16).astype(np.float64)
    assert es.abs_value == 2 * sum(Fraction(v) for v in pos.tolist())


def test_empty_is_zero(spec_golden):
    es = oracle.exact_sum_fp16(np.zeros(0, dtype=np.uint16))
    assert es.T == 0 and es.A == 0 and es.f32() == 0.0


def test_arithmetic_series(spec_golden):
    x = np.arange(1, 17, dtype=np.float16)
    assert oracle.exact_sum_fp16(x).value == 136
    k = 2048  # integers up to 2048 are exact in binary16
    x = np.arange(1, k + 1, dtype=np.float16)
    assert oracle.exact_sum_fp16(x).value == k * (k + 1) // 2


def test_all_ones_gives_n():
    n = (1 << 20) + 7
    x = gen.generate(0, 0, n, gen.ONES)
    es = oracle.exact_sum_fp16(x)
    assert es.value == n and es.abs_value == n


def test_alternating_cancels_to_zero():
    n = 100_002
    x = gen.generate(gen.SEED_C1, 0, n, gen.ALTERNATING)
    es = oracle.exact_sum_fp16(x)
    assert es.T == 0
    assert es.A > 0


@pytest.mark.parametrize("dist", [gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01, gen.SMALLINT])
def test_brute_force_fraction_tiny(dist):
    for seed in range(5):
        for n in (1, 2, 3, 7, 31, 256, 257, 1000):
            x = gen.generate(seed, 17 * seed, n, dist)
            assert oracle.exact_sum_fp16(x).value == oracle.exact_sum_fraction(x)


def test_fsum_correctly_rounded_matches():
    # math.fsum returns the correctly rounded binary64 sum of binary64 inputs.
    for dist in (gen.UNIFORM_PM1, gen.WIDE):
        x = gen.generate(99, 0, 200_000, dist)
        es = oracle.exact_sum_fp16(x)
        assert es.f64() == math.fsum(x.view(np.float16).astype(np.float64).tolist())


def test_overflow_headroom_beyond_int64():
    # |x| = 65504 at n > 2^23 overflows a single int64 in 2^-24 units; int128 does not.
    n = (1 << 24) + 5
    x = np.full(n, np.float16(65504.0)).view(np.uint16)
    es = oracle.exact_sum_fp16(x, threads=4)
    assert es.value == n * 65504
    assert es.T > (1 << 63)


def test_thread_count_invariance_and_homomorphism():
    x = gen.generate(7, 0, 1_000_003, gen.WIDE)
    ref = oracle.exact_sum_fp16(x, threads=1)
    for t in (2, 3, 7, 8):
        assert oracle.exact_sum_fp16(x, threads=t) == ref
    k = 123_457
    assert oracle.exact_sum_fp16(x[:k]) + oracle.exact_sum_fp16(x[k:]) == ref


def test_permutation_invariance():
    x = gen.generate(3, 0, 50_000, gen.WIDE)
    rng = np.random.default_rng(0)
    assert oracle.exact_sum_fp16(rng.permutation(x)) == oracle.exact_sum_fp16(x)


def test_specials():
    one, pinf, ninf, nan = 0x3C00, 0x7C00, 0xFC00, 0x7E00
    s = lambda *v: oracle.exact_sum_fp16(np.array(v, dtype=np.uint16)).f32()
    assert s(one, pinf) == math.inf
    assert s(one, ninf) == -math.inf
    assert math.isnan(s(pinf, ninf))
    assert math.isnan(s(one, nan))
    es = oracle.exact_sum_fp16(np.array([one, pinf], dtype=np.uint16))
    assert oracle.within_tolerance(math.inf, es) and not oracle.within_tolerance(1.0, es)


def test_segments_match_slices_and_reject_decreasing():
    x = gen.generate(5, 0, 10_000, gen.WIDE)
    off = np.array([0, 0, 1, 100, 4097, 4097, 10_000], dtype=np.int64)
    res = oracle.exact_segment_sums_fp16(x, off)
    for j in range(len(off) - 1):
        assert res[j] == oracle.exact_sum_fp16(x[off[j]:off[j + 1]])
    with pytest.raises(ValueError):
        oracle.exact_segment_sums_fp16(x, np.array([0, 10, 5], dtype=np.int64))


def test_round_to_f32_matches_numpy_for_doubles():
    # numpy's float64 -> float32 cast is IEEE RNE; a double is an exact rational.
    rng = np.random.default_rng(1)
    vals = np.concatenate([
        rng.standard_normal(20_000) * np.exp2(rng.integers(-140, 120, 20_000)),
        np.array([1 + 2.0 ** -24, 1 + 3 * 2.0 ** -24, 1 + 2.0 ** -23 + 2.0 ** -24,  # ties
                  2.0 ** -149, 2.0 ** -150, 3 * 2.0 ** -150, 2.0 ** -126 * (1 - 2.0 ** -24),
                  3.4028235677973366e38, 3.4028235677973362e38 * (1 + 2.0 ** -25)]),
    ])
    with np.errstate(over="ignore"):  # values past FLT_MAX round to inf, on purpose
        for v in vals.tolist():
            assert oracle.round_to_f32(Fraction(v)) == float(np.float32(v)), v


def test_within_tolerance_boundary_is_exact():
    x = gen.generate(11, 0, 4096, gen.UNIFORM_01)
    es = oracle.exact_sum_fp16(x)
    tol = es.abs_value / (1 << 20)
    R = es.value
    # construct binary32 values just inside / outside the bound
    inside = float(np.float32(float(R + tol * Fraction(9, 10))))
    assert abs(Fraction(inside) - R) <= tol
    assert oracle.within_tolerance(inside, es)
    outside = float(np.nextafter(np.float32(float(R + tol)), np.float32(np.inf)))
    assert abs(Fraction(outside) - R) > tol
    assert not oracle.within_tolerance(outside, es)
    assert oracle.within_tolerance(es.f32(), es)


def test_generator_rne_matches_struct_half_pack(spec_golden):
    # Independent binary16 RNE: struct's 'e' format packs a double with round-half-even.
    for ex in spec_golden["quantize_fp16"]:
        assert struct.unpack("<e", struct.pack("<e", ex["v"]))[0] == ex["fp16"]
        assert float(np.float16(ex["v"])) == ex["fp16"]
    idx = np.arange(0, 5000, dtype=np.uint64)
    z = gen.splitmix64(gen.SEED_C1, idx)
    bits = gen.generate(gen.SEED_C1, 0, 5000, gen.UNIFORM_PM1)
    for zi, b in zip(z.tolist(), bits.tolist()):
        v = (zi >> 40) * 2.0 ** -23 - 1.0
        assert -1.0 <= v < 1.0
        ref = struct.unpack("<H", struct.pack("<e", v))[0]
        assert ref == b


def test_generator_shard_invariance():
    full = gen.generate(gen.SEED_C4, 1000, 4096, gen.UNIFORM_PM1)
    a = gen.generate(gen.SEED_C4, 1000, 1500, gen.UNIFORM_PM1)
    b = gen.generate(gen.SEED_C4, 2500, 2596, gen.UNIFORM_PM1)
    assert np.array_equal(full, np.concatenate([a, b]))


def test_loguniform_lengths_recipe():
    L = gen.loguniform_lengths(gen.SEED_C5, 1 << 16)
    assert L.min() >= 256 and L.max() <= 65536
    # mean of a log-uniform integer on [256, 65536] ~ (65536-256)/ln(256) ~ 11.8k
    assert 11_000 < L.mean() < 12_600
    off = gen.offsets_from_lengths(L)
    assert off[0] == 0 and np.all(np.diff(off) == L)
