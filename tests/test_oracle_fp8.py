"""Pins for the fp8 (E4M3 / E5M2) oracle and generator (NEXT-4), CPU only:
torch's float8 decoding and float32 -> float8 RNE conversion (an independent
implementation), Python Fractions, math.fsum, closed forms, invariants."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

torch = pytest.importorskip("torch")
FMTS = {oracle.FP8_E4M3: torch.float8_e4m3fn, oracle.FP8_E5M2: torch.float8_e5m2}


def _finite(fmt):
    bits = np.arange(256, dtype=np.uint8)
    vals = torch.from_numpy(bits).view(FMTS[fmt]).float().numpy()
    return bits[np.isfinite(vals)], vals[np.isfinite(vals)].astype(np.float64)


@pytest.mark.parametrize("fmt", [oracle.FP8_E4M3, oracle.FP8_E5M2])
def test_decode_all_patterns_vs_torch(fmt):
    bits, vals = _finite(fmt)
    assert len(bits) == (254 if fmt == oracle.FP8_E4M3 else 248)
    for b, v in zip(bits.tolist(), vals.tolist()):
        assert oracle.fp8_value(b, fmt) == Fraction(v)
        assert oracle.exact_sum_fp8(np.array([b], np.uint8), fmt).value == Fraction(v)


@pytest.mark.parametrize("fmt", [oracle.FP8_E4M3, oracle.FP8_E5M2])
def test_sums_brute_force_fsum_closed_forms(fmt):
    for seed in range(3):
        for dist in (gen.WIDE, gen.UNIFORM_PM1, gen.SMALLINT):
            x = gen.generate_fp8(seed, 3 * seed, 999, dist, fmt)
            ref = sum((oracle.fp8_value(int(b), fmt) for b in x.tolist()), Fraction(0))
            assert oracle.exact_sum_fp8(x, fmt).value == ref
    x = gen.generate_fp8(4, 0, 200_000, gen.WIDE, fmt)
    vals = torch.from_numpy(x).view(FMTS[fmt]).double().numpy()
    assert oracle.exact_sum_fp8(x, fmt).f64() == math.fsum(vals.tolist())
    assert oracle.exact_sum_fp8(gen.generate_fp8(0, 0, 1001, gen.ONES, fmt), fmt).value == 1001
    assert oracle.exact_sum_fp8(gen.generate_fp8(1, 0, 5000, gen.ALTERNATING, fmt), fmt).T == 0


@pytest.mark.parametrize("fmt", [oracle.FP8_E4M3, oracle.FP8_E5M2])
def test_generator_rne_matches_torch(fmt):
    idx = np.arange(0, 100_000, dtype=np.uint64)
    z = gen.splitmix64(gen.SEED_C1, idx)
    for dist, sc, off in ((gen.UNIFORM_PM1, 2.0 ** -23, 1.0), (gen.UNIFORM_01, 2.0 ** -24, 0.0)):
        v = (z >> np.uint64(40)).astype(np.float32) * np.float32(sc) - np.float32(off)
        ref = torch.from_numpy(v).to(FMTS[fmt]).view(torch.uint8).numpy()
        assert np.array_equal(gen.generate_fp8(gen.SEED_C1, 0, 100_000, dist, fmt), ref)


def test_specials():
    s8 = lambda fmt, *b: oracle.exact_sum_fp8(np.array(b, np.uint8), fmt).f32()
    assert math.isnan(s8(oracle.FP8_E4M3, 0x38, 0x7F))
    assert s8(oracle.FP8_E5M2, 0x3C, 0x7C) == math.inf and s8(oracle.FP8_E5M2, 0xFC) == -math.inf
    assert math.isnan(s8(oracle.FP8_E5M2, 0x7C, 0xFC))
