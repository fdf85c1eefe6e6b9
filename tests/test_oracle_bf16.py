"""Pins for the bfloat16 oracle and generator (NEXT-4), CPU only.

Checked against numpy's binary32 decoding of (bits << 16) (bfloat16 is the
top half of a binary32), Python Fractions, math.fsum, torch's CPU
float32 -> bfloat16 conversion, and invariants.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

ALL_FINITE = np.array([h for h in range(1 << 16) if ((h >> 7) & 0xFF) != 0xFF], dtype=np.uint16)


def _f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_decode_all_finite_patterns():
    vals = _f64(ALL_FINITE).tolist()
    for h, v in zip(ALL_FINITE.tolist()[::7], vals[::7]):
        assert oracle.bf16_value(h) == Fraction(v)
    # the bins oracle on single elements
    for h in ALL_FINITE.tolist()[::97]:
        es = oracle.exact_sum_bf16(np.array([h], dtype=np.uint16))
        assert es.value == oracle.bf16_value(h)


def test_sum_of_all_patterns_and_brute_force():
    es = oracle.exact_sum_bf16(ALL_FINITE)
    assert es.T == 0  # symmetric
    for seed in range(4):
        for dist in (gen.WIDE, gen.UNIFORM_PM1, gen.SMALLINT):
            x = gen.generate_bf16(seed, 11 * seed, 777, dist)
            ref = sum((Fraction(v) for v in _f64(x).tolist()), Fraction(0))
            assert oracle.exact_sum_bf16(x).value == ref


def test_fsum_and_closed_forms():
    x = gen.generate_bf16(5, 0, 300_000, gen.WIDE)
    es = oracle.exact_sum_bf16(x)
    assert es.f64() == math.fsum(_f64(x).tolist())
    n = 100_003
    assert oracle.exact_sum_bf16(gen.generate_bf16(0, 0, n, gen.ONES)).value == n
    assert oracle.exact_sum_bf16(gen.generate_bf16(1, 0, 100_000, gen.ALTERNATING)).T == 0


def test_homomorphism_permutation_specials():
    x = gen.generate_bf16(9, 0, 50_001, gen.WIDE)
    es = oracle.exact_sum_bf16(x)
    assert oracle.exact_sum_bf16(x[:123]) + oracle.exact_sum_bf16(x[123:]) == es
    assert oracle.exact_sum_bf16(np.random.default_rng(0).permutation(x)) == es
    s = lambda *v: oracle.exact_sum_bf16(np.array(v, dtype=np.uint16)).f32()
    assert s(0x3F80, 0x7F80) == math.inf and s(0x3F80, 0xFF80) == -math.inf
    assert math.isnan(s(0x7F80, 0xFF80)) and math.isnan(s(0x7FC1))


def test_bf16_generator_matches_torch_rne():
    torch = pytest.importorskip("torch")
    idx = np.arange(0, 20_000, dtype=np.uint64)
    for dist, scale, off in ((gen.UNIFORM_PM1, 2.0 ** -23, 1.0), (gen.UNIFORM_01, 2.0 ** -24, 0.0)):
        z = gen.splitmix64(gen.SEED_C1, idx)
        v = (z >> np.uint64(40)).astype(np.float32) * np.float32(scale) - np.float32(off)
        ref = torch.from_numpy(v).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(gen.generate_bf16(gen.SEED_C1, 0, 20_000, dist), ref)
    assert np.array_equal(gen.f32_to_bf16_rne(np.array([1.0 + 2.0 ** -8], np.float32)),
                          np.array([0x3F80], np.uint16))  # tie -> even
    assert np.array_equal(gen.f32_to_bf16_rne(np.array([1.0 + 3 * 2.0 ** -8], np.float32)),
                          np.array([0x3F82], np.uint16))  # tie -> even (up)
