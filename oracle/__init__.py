"""oracle -- TEST INFRASTRUCTURE ONLY (never on the product path).

The exact CPU oracle for arXiv 1903.03640 ("Analyzing GPU Tensor Core
Potential for Fast Reductions").  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import
this package.  It shares no code, header, table or constant with the CUDA
path in ``paper_1903_03640_b200/`` and never imports it.

Contents
--------
* :func:`exact_sum_fp16` -- R(X) = sum x_i exactly (§III Eq. 2,
  lines 106-110), via the plain C loop in ``exact_sum.c`` (int128 in units of
  2^-24).  Also returns A = sum |x_i| exactly.
* :func:`exact_sum_fraction` -- the same definition in pure Python
  ``fractions.Fraction`` arithmetic, for tiny inputs (an independent check of
  the C code).
* :func:`exact_segment_sums_fp16_array` / ``_fp8_array`` / :func:`exact_segment_sums_bf16`
  -- the same per segment of a CSR partition, for large segment counts, and
  :func:`within_tolerance_segments`, the acceptance test over all of them.
* :func:`within_tolerance` -- the north-star acceptance test
  |g - R| <= 2^-20 * sum|x_i|, evaluated in exact rational arithmetic
  (reading G15).
* :func:`round_to_f32` -- correctly rounded (RNE) binary32 of an exact value.
* :mod:`oracle.model` -- the paper's structural algorithm R_tc (Eq. 9-14)
  in exact arithmetic and its cost model (Eq. 15-17).

Pins: every function here is pinned by ``tests/test_oracle_*.py`` against
closed forms, invariants, brute force and the paper's printed values
(see DESIGN.md §"Oracle and pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC_PATH = os.path.join(_HERE, "exact_sum.c")

UNIT = Fraction(1, 1 << 24)  # every finite binary16 value is a multiple of 2^-24


class _Result(ctypes.Structure):
    _fields_ = [
        ("t_lo", ctypes.c_uint64),
        ("t_hi", ctypes.c_int64),
        ("a_lo", ctypes.c_uint64),
        ("a_hi", ctypes.c_uint64),
        ("n_nan", ctypes.c_uint64),
        ("n_pinf", ctypes.c_uint64),
        ("n_ninf", ctypes.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile ``exact_sum.c`` into ``liboracle.so`` with gcc (plain -O2)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC_PATH)
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.run(
            ["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC_PATH],
            check=True,
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_exact_sum_fp16.argtypes = [
            ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(_Result)]
        lib.oracle_exact_sum_fp16.restype = ctypes.c_int
        lib.oracle_exact_segment_sums_fp16.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.oracle_exact_segment_sums_fp16.restype = ctypes.c_int
        lib.oracle_exact_bins_bf16.argtypes = [
            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_exact_bins_bf16.restype = ctypes.c_int
        lib.oracle_exact_sum_fp8.argtypes = [
            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(_Result)]
        lib.oracle_exact_sum_fp8.restype = ctypes.c_int
        lib.oracle_exact_segment_sums_fp8.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
        lib.oracle_exact_segment_sums_fp8.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass(frozen=True)
class ExactSum:
    """Exact result of R(X): T = sum x_i / unit and A = sum |x_i| / unit (ints).

    unit = 2^unit_exp: 2^-24 for binary16 inputs, 2^-133 for bfloat16.
    """

    T: int
    A: int
    n_nan: int = 0
    n_pinf: int = 0
    n_ninf: int = 0
    unit_exp: int = -24

    def __add__(self, other: "ExactSum") -> "ExactSum":
        # Exact homomorphism R(X ++ Y) = R(X) + R(Y).
        if self.unit_exp != other.unit_exp:
            raise ValueError("cannot add sums in different units")
        return ExactSum(self.T + other.T, self.A + other.A, self.n_nan + other.n_nan,
                        self.n_pinf + other.n_pinf, self.n_ninf + other.n_ninf, self.unit_exp)

    @property
    def unit(self) -> Fraction:
        return Fraction(2) ** self.unit_exp

    @property
    def finite(self) -> bool:
        return self.n_nan == 0 and self.n_pinf == 0 and self.n_ninf == 0

    @property
    def special(self) -> float | None:
        """IEEE propagation for non-finite inputs (reading G13)."""
        if self.n_nan or (self.n_pinf and self.n_ninf):
            return float("nan")
        if self.n_pinf:
            return float("inf")
        if self.n_ninf:
            return float("-inf")
        return None

    @property
    def value(self) -> Fraction:
        """R(X) as an exact rational."""
        return self.T * self.unit

    @property
    def abs_value(self) -> Fraction:
        return self.A * self.unit

    def f32(self) -> float:
        """Correctly rounded (RNE) binary32 value of R(X), as a Python float."""
        s = self.special
        return s if s is not None else round_to_f32(self.value)

    def f64(self) -> float:
        """Correctly rounded binary64 value of R(X) (Fraction.__float__ is RNE)."""
        s = self.special
        return s if s is not None else float(self.value)


def _from_struct(r: _Result) -> ExactSum:
    t = (int(r.t_hi) << 64) | int(r.t_lo)
    a = (int(r.a_hi) << 64) | int(r.a_lo)
    return ExactSum(t, a, int(r.n_nan), int(r.n_pinf), int(r.n_ninf))


def _as_bits(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype == np.float16:
        x = x.view(np.uint16)
    if x.dtype != np.uint16:
        raise TypeError(f"expected binary16 bit patterns (uint16/float16), got {x.dtype}")
    return np.ascontiguousarray(x.reshape(-1))


def exact_sum_fp16(x, threads: int = 1) -> ExactSum:
    """Exact R(X) (Eq. 2) of binary16 inputs ``x`` (uint16 bits or float16).

    ``threads`` > 1 splits X into contiguous chunks reduced concurrently and
    adds the exact chunk results (homomorphism); the result is
    identical for every thread count because integer addition is exact.
    """
    bits = _as_bits(x)
    lib = _load()
    n = bits.size
    threads = max(1, min(int(threads), max(1, n)))

    def run(lo: int, hi: int) -> ExactSum:
        r = _Result()
        lib.oracle_exact_sum_fp16(bits.ctypes.data + 2 * lo, hi - lo, ctypes.byref(r))
        return _from_struct(r)

    if threads == 1:
        return run(0, n)
    bounds = [n * k // threads for k in range(threads + 1)]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(lambda k: run(bounds[k], bounds[k + 1]), range(threads)))
    total = ExactSum(0, 0)
    for p in parts:
        total = total + p
    return total


def exact_segment_sums_fp16(x, offsets) -> list[ExactSum]:
    """Exact per-segment R for CSR ``offsets`` (segment j = x[off[j]:off[j+1]])."""
    bits = _as_bits(x)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    s = off.size - 1
    if s < 0:
        raise ValueError("offsets must hold num_segments + 1 entries")
    if s and (off[0] < 0 or off[-1] > bits.size):
        raise ValueError("offsets out of range")
    res = (_Result * max(s, 1))()
    rc = _load().oracle_exact_segment_sums_fp16(bits.ctypes.data, off.ctypes.data, s,
                                                ctypes.addressof(res))
    if rc != 0:
        raise ValueError("offsets must be non-decreasing")
    return [_from_struct(res[j]) for j in range(s)]


# numpy view of an array of oracle_sum_result records (exact_sum.c)
_REC_DTYPE = np.dtype([("t_lo", "<u8"), ("t_hi", "<i8"), ("a_lo", "<u8"), ("a_hi", "<u8"),
                       ("n_nan", "<u8"), ("n_pinf", "<u8"), ("n_ninf", "<u8")])


class SegmentSums:
    """Exact per-segment R(X_j) for many segments, held as the C oracle's
    records (int128 T and A per segment, in units of 2^unit_exp) rather than
    one Python object per segment; ``ss[j]`` is the segment's ExactSum."""

    def __init__(self, rec: np.ndarray, unit_exp: int):
        self.rec = rec
        self.unit_exp = unit_exp

    def __len__(self) -> int:
        return self.rec.size

    def __getitem__(self, j: int) -> ExactSum:
        r = self.rec[j]
        t = (int(r["t_hi"]) << 64) | int(r["t_lo"])
        a = (int(r["a_hi"]) << 64) | int(r["a_lo"])
        return ExactSum(t, a, int(r["n_nan"]), int(r["n_pinf"]), int(r["n_ninf"]), self.unit_exp)


def _segment_records(fn, bits, off, threads, *extra) -> np.ndarray:
    """Call the C per-segment loop ``fn`` over contiguous ranges of segments
    (one range per thread; the records do not depend on the split)."""
    s = off.size - 1
    rec = np.zeros(max(s, 1), dtype=_REC_DTYPE)
    threads = max(1, min(int(threads), max(1, s)))
    bounds = [s * k // threads for k in range(threads + 1)]

    def run(k: int) -> int:
        j0, j1 = bounds[k], bounds[k + 1]
        return fn(bits.ctypes.data, off.ctypes.data + 8 * j0, j1 - j0, *extra,
                  rec.ctypes.data + rec.itemsize * j0)

    if threads == 1:
        rcs = [run(0)]
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            rcs = list(ex.map(run, range(threads)))
    if any(rcs):
        raise ValueError("offsets must be non-decreasing")
    return rec[:s]


def _check_offsets(off: np.ndarray, size: int) -> None:
    if off.size < 1:
        raise ValueError("offsets must hold num_segments + 1 entries")
    if off.size > 1 and (off[0] < 0 or off[-1] > size):
        raise ValueError("offsets out of range")


def exact_segment_sums_fp16_array(x, offsets, threads: int = 1) -> SegmentSums:
    """Exact per-segment R for CSR ``offsets`` of binary16 inputs, as records
    (same C loop as :func:`exact_segment_sums_fp16`), for large S."""
    bits = _as_bits(x)
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    _check_offsets(off, bits.size)
    return SegmentSums(_segment_records(_load().oracle_exact_segment_sums_fp16, bits, off, threads),
                       -24)


def exact_segment_sums_fp8_array(x, offsets, fmt: int, threads: int = 1) -> SegmentSums:
    """Exact per-segment R of fp8 bit patterns (uint8) for CSR ``offsets``."""
    bits = np.ascontiguousarray(np.asarray(x, dtype=np.uint8).reshape(-1))
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    _check_offsets(off, bits.size)
    rec = _segment_records(_load().oracle_exact_segment_sums_fp8, bits, off, threads, int(fmt))
    return SegmentSums(rec, _FP8_UNIT_EXP[fmt])


def exact_segment_sums_bf16(x, offsets) -> list[ExactSum]:
    """Exact per-segment R of bfloat16 bit patterns: :func:`exact_sum_bf16`
    applied to each segment x[off[j]:off[j+1]]."""
    bits = np.ascontiguousarray(np.asarray(x, dtype=np.uint16).reshape(-1))
    off = np.asarray(offsets, dtype=np.int64)
    _check_offsets(off, bits.size)
    if np.any(np.diff(off) < 0):
        raise ValueError("offsets must be non-decreasing")
    return [exact_sum_bf16(bits[int(off[j]):int(off[j + 1])]) for j in range(off.size - 1)]


def exact_sum_bf16(x) -> ExactSum:
    """Exact R(X) of bfloat16 bit patterns (uint16) -- NEXT-4.

    The C loop bins the integer significands by exponent (``exact_sum.c``);
    the bins are combined here in Python integers: T = sum_e bin[e] *
    2^max(e-1, 0) in units of 2^-133 (exact, no overflow).
    """
    bits = np.ascontiguousarray(np.asarray(x, dtype=np.uint16).reshape(-1))
    bins = np.zeros(256, dtype=np.int64)
    abins = np.zeros(256, dtype=np.uint64)
    counts = np.zeros(3, dtype=np.uint64)
    _load().oracle_exact_bins_bf16(bits.ctypes.data, bits.size, bins.ctypes.data,
                                   abins.ctypes.data, counts.ctypes.data)
    # bins with no inputs contribute nothing: only the occupied exponents are visited
    used = np.nonzero(abins)[0].tolist()
    T = sum(int(bins[e]) << max(e - 1, 0) for e in used)
    A = sum(int(abins[e]) << max(e - 1, 0) for e in used)
    return ExactSum(T, A, int(counts[0]), int(counts[1]), int(counts[2]), unit_exp=-133)


FP8_E4M3, FP8_E5M2 = 0, 1
_FP8_UNIT_EXP = {FP8_E4M3: -9, FP8_E5M2: -16}


def exact_sum_fp8(x, fmt: int) -> ExactSum:
    """Exact R(X) of fp8 bit patterns (uint8): fmt 0 = E4M3 (units 2^-9),
    fmt 1 = E5M2 (units 2^-16) -- NEXT-4.  Plain loop in ``exact_sum.c``."""
    bits = np.ascontiguousarray(np.asarray(x, dtype=np.uint8).reshape(-1))
    r = _Result()
    _load().oracle_exact_sum_fp8(bits.ctypes.data, bits.size, int(fmt), ctypes.byref(r))
    es = _from_struct(r)
    return ExactSum(es.T, es.A, es.n_nan, es.n_pinf, es.n_ninf, unit_exp=_FP8_UNIT_EXP[fmt])


def fp8_value(h: int, fmt: int) -> Fraction:
    """Exact value of one finite fp8 bit pattern, from the OCP FP8 definition."""
    eb, mb, bias = (4, 3, 7) if fmt == FP8_E4M3 else (5, 2, 15)
    s, e, f = (h >> 7) & 1, (h >> mb) & ((1 << eb) - 1), h & ((1 << mb) - 1)
    if (fmt == FP8_E4M3 and e == 15 and f == 7) or (fmt == FP8_E5M2 and e == 31):
        raise ValueError("non-finite")
    if e == 0:
        v = Fraction(f, 1 << mb) * Fraction(2) ** (1 - bias)
    else:
        v = (1 + Fraction(f, 1 << mb)) * Fraction(2) ** (e - bias)
    return -v if s else v


def bf16_value(h: int) -> Fraction:
    """Exact value of one finite bfloat16 bit pattern, from the definition."""
    s, e, f = (h >> 15) & 1, (h >> 7) & 0xFF, h & 0x7F
    if e == 0xFF:
        raise ValueError("non-finite")
    v = Fraction(f, 128) * Fraction(2) ** -126 if e == 0 else (1 + Fraction(f, 128)) * Fraction(2) ** (e - 127)
    return -v if s else v


def exact_sum_fraction(values) -> Fraction:
    """Pure-Python exact sum of binary16 inputs (brute force for tiny n).

    Each element is converted by numpy to float64 (exact for binary16) and
    then to ``Fraction`` (exact), and the Fractions are added left to right.
    Independent of ``exact_sum.c``.
    """
    f = np.asarray(values)
    if f.dtype == np.uint16:
        f = f.view(np.float16)
    total = Fraction(0)
    for v in f.astype(np.float64).tolist():
        total += Fraction(v)
    return total


def round_to_f32(q: Fraction) -> float:
    """Round an exact rational to binary32, round-to-nearest-even.

    Returns a Python float holding the binary32 value exactly (inf on
    overflow).  Written from the IEEE-754 definition: quantum 2^(e-23) for
    normal exponents e >= -126, 2^-149 below; ties to the even significand.
    """
    q = Fraction(q)
    if q == 0:
        return 0.0
    sign = -1.0 if q < 0 else 1.0
    a = abs(q)
    # e = floor(log2(a)), exactly.
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    quantum = Fraction(2) ** (max(e, -126) - 23)
    m = a / quantum
    mi = m.numerator // m.denominator
    rem = m - mi
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and (mi & 1)):
        mi += 1
    r = mi * quantum
    if r >= Fraction(2) ** 128:
        return sign * float("inf")
    return sign * float(r)


def within_tolerance(g: float, es: ExactSum, rel: Fraction = Fraction(1, 1 << 20)) -> bool:
    """North-star acceptance test, exact: |g - R(X)| <= rel * sum |x_i|.

    ``g`` is the GPU's binary32 (or binary64) result.  Non-finite expected
    values must match exactly (NaN matches NaN).  Evaluated in rationals, so
    there is no rounding ambiguity at the boundary (reading G15).
    """
    s = es.special
    if s is not None:
        if s != s:
            return g != g
        return g == s
    if not np.isfinite(g):
        return False
    return abs(Fraction(float(g)) - es.value) <= rel * es.abs_value


def within_tolerance_segments(g, ss: SegmentSums, rel_log2: int = 20) -> np.ndarray:
    """:func:`within_tolerance` for every segment: ok[j] iff
    |g[j] - R_j| <= 2^-rel_log2 * sum|x| over segment j.

    Where T_j, A_j and G_j = g[j] / unit are integers below 2^62 (always, for
    the configs' fp16 / fp8 segments) the test is the same exact integer
    comparison |G - T| * 2^rel <= A, written as |G - T| <= floor(A / 2^rel)
    (equivalent for integer |G - T|) and evaluated on int64 arrays; every
    other segment (specials, g not a multiple of the unit, larger values)
    goes through the scalar rational :func:`within_tolerance`.
    """
    g = np.asarray(g, dtype=np.float64).reshape(-1)
    rec = ss.rec
    if g.size != rec.size:
        raise ValueError("one result per segment expected")
    lim = np.uint64(1 << 62)
    t_lo_s = rec["t_lo"].view(np.int64)
    fits = ((rec["t_hi"] == (t_lo_s >> 63)) & (np.abs(t_lo_s) < (1 << 62))
            & (rec["a_hi"] == 0) & (rec["a_lo"] < lim)
            & (rec["n_nan"] == 0) & (rec["n_pinf"] == 0) & (rec["n_ninf"] == 0))
    with np.errstate(invalid="ignore", over="ignore"):
        G = np.ldexp(g, -ss.unit_exp)  # exact: scaling by a power of two
        fits &= np.isfinite(G) & (np.abs(G) < 2.0 ** 62) & (G == np.floor(G))
    ok = np.zeros(g.size, dtype=bool)
    idx = np.nonzero(fits)[0]
    Gi = G[idx].astype(np.int64)
    diff = np.abs(Gi - t_lo_s[idx])
    ok[idx] = diff <= (rec["a_lo"][idx] >> np.uint64(rel_log2)).astype(np.int64)
    for j in np.nonzero(~fits)[0].tolist():
        ok[j] = within_tolerance(float(g[j]), ss[j], Fraction(1, 1 << rel_log2))
    return ok


def error_units(g: float, es: ExactSum) -> Fraction:
    """|g - R(X)| in units of 2^-24 (exact, for every input type: the unit is
    fixed at 2^-24, not the type's own quantum)."""
    return abs(Fraction(float(g)) - es.value) / UNIT


__all__ = [
    "ExactSum", "UNIT", "build", "exact_sum_fp16", "exact_segment_sums_fp16", "exact_sum_bf16",
    "bf16_value", "exact_sum_fp8", "fp8_value", "FP8_E4M3", "FP8_E5M2",
    "exact_sum_fraction", "round_to_f32", "within_tolerance", "error_units",
    "SegmentSums", "exact_segment_sums_fp16_array", "exact_segment_sums_fp8_array",
    "exact_segment_sums_bf16", "within_tolerance_segments",
]
