/*
 * oracle/exact_sum.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The exact CPU oracle for the sum reduction of arXiv 1903.03640.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this file's library.  The product path
 * (paper_1903_03640_b200/) never links, imports or calls it, and this file
 * shares no code, header or constant with the CUDA path.
 *
 * What it computes (§III, Eq. 2):
 *
 *     R(X) = sum_{i=1..n} x_i
 *
 * exactly, for x_i IEEE-754 binary16 values.  Every finite binary16 value is
 * an integer multiple of 2^-24 with magnitude below 2^16 (so |x_i * 2^24|
 * < 2^40).  The oracle therefore represents each x_i as the integer
 * u_i = x_i * 2^24 and adds the u_i in a signed 128-bit integer: for any
 * n < 2^87 the sum cannot overflow, and integer addition is exact and
 * independent of order.  This is the plain definition of Eq. 2 written out,
 * with no blocking, reordering or rounding.
 *
 * Decoding (IEEE-754 binary16): s = bit 15, e = bits 14..10, f = bits 9..0.
 *     e == 0          : value = (-1)^s * f * 2^-24          -> u = f
 *     1 <= e <= 30    : value = (-1)^s * (1024+f) * 2^(e-25) -> u = (1024+f) << (e-1)
 *     e == 31, f == 0 : +/- infinity (flag)
 *     e == 31, f != 0 : NaN (flag)
 *
 * It also returns A = sum |x_i| * 2^24 exactly (the tolerance scale of the
 * north star: |gpu - R| <= 2^-20 * sum |x_i|).
 *
 * Build: gcc -O2 -std=c11 -shared -fPIC -o liboracle.so exact_sum.c
 * (done by oracle.build(), called from __graft_entry__.build()).
 */
#include <stddef.h>
#include <stdint.h>

typedef __int128 i128;
typedef unsigned __int128 u128;

/* Result record, returned through a caller-owned struct (ctypes-friendly). */
typedef struct {
    uint64_t t_lo;   /* T = sum u_i as two's-complement int128: low 64 bits  */
    int64_t  t_hi;   /*                                         high 64 bits */
    uint64_t a_lo;   /* A = sum |u_i| as unsigned int128: low 64 bits        */
    uint64_t a_hi;   /*                                    high 64 bits      */
    uint64_t n_nan;  /* number of NaN inputs                                 */
    uint64_t n_pinf; /* number of +inf inputs                                */
    uint64_t n_ninf; /* number of -inf inputs                                */
} oracle_sum_result;

/* Value of one binary16 bit pattern in units of 2^-24 (finite inputs only). */
static i128 fp16_units(uint16_t h) {
    const unsigned s = (h >> 15) & 1u;
    const unsigned e = (h >> 10) & 0x1fu;
    const unsigned f = h & 0x3ffu;
    i128 u;
    if (e == 0) {
        u = (i128)f;                              /* subnormal or zero */
    } else {
        u = (i128)(1024u + f) << (e - 1);         /* normal */
    }
    return s ? -u : u;
}

/*
 * Exact sum of x[0..n).  Writes *r.  Returns 0.
 * Non-finite inputs are counted in the flags and excluded from T and A;
 * the caller applies IEEE propagation (reading G13).
 */
int oracle_exact_sum_fp16(const uint16_t *x, size_t n, oracle_sum_result *r) {
    i128 t = 0;
    u128 a = 0;
    uint64_t n_nan = 0, n_pinf = 0, n_ninf = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint16_t h = x[i];
        if (((h >> 10) & 0x1fu) == 0x1fu) {       /* e == 31: inf or NaN */
            if (h & 0x3ffu) {
                ++n_nan;
            } else if (h >> 15) {
                ++n_ninf;
            } else {
                ++n_pinf;
            }
            continue;
        }
        const i128 u = fp16_units(h);
        t += u;
        a += (u128)(u < 0 ? -u : u);
    }
    r->t_lo = (uint64_t)(u128)t;
    r->t_hi = (int64_t)(t >> 64);
    r->a_lo = (uint64_t)a;
    r->a_hi = (uint64_t)(a >> 64);
    r->n_nan = n_nan;
    r->n_pinf = n_pinf;
    r->n_ninf = n_ninf;
    return 0;
}

/*
 * Exact per-segment sums (CSR): segment j is x[offsets[j] .. offsets[j+1]).
 * Writes one record per segment into r[0..num_segments).  offsets must be
 * non-decreasing with offsets[num_segments] <= the length of x.
 * Returns 0, or -1 if the offsets are decreasing (nothing written past j).
 */
int oracle_exact_segment_sums_fp16(const uint16_t *x, const int64_t *offsets,
                                   size_t num_segments, oracle_sum_result *r) {
    for (size_t j = 0; j < num_segments; ++j) {
        if (offsets[j + 1] < offsets[j]) return -1;
        oracle_exact_sum_fp16(x + offsets[j], (size_t)(offsets[j + 1] - offsets[j]), &r[j]);
    }
    return 0;
}

/*
 * bfloat16 (NEXT-4): value = (-1)^s * 2^(e-127) * (1 + f/128) for
 * 1 <= e <= 254, (-1)^s * f * 2^-133 for e == 0; every finite bfloat16 is
 * an integer multiple of 2^-133 below 2^128, so the exact sum needs ~262
 * bits.  The oracle keeps, per biased exponent e, the signed sum of the
 * integer significands sig = (e == 0 ? f : 128 + f) < 2^8 in an int64 bin
 * (safe for n < 2^55) and the sum of |sig|; the caller forms
 * T = sum_e bin[e] * 2^max(e-1, 0) in arbitrary precision (units 2^-133).
 * bins / abs_bins: caller-owned int64[256] / uint64[256], overwritten.
 * counts[3] = NaN, +inf, -inf inputs.
 */
int oracle_exact_bins_bf16(const uint16_t *x, size_t n, int64_t *bins, uint64_t *abs_bins,
                           uint64_t *counts) {
    for (int e = 0; e < 256; ++e) {
        bins[e] = 0;
        abs_bins[e] = 0;
    }
    counts[0] = counts[1] = counts[2] = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint16_t h = x[i];
        const unsigned s = (h >> 15) & 1u;
        const unsigned e = (h >> 7) & 0xffu;
        const unsigned f = h & 0x7fu;
        if (e == 0xffu) {
            if (f) ++counts[0];
            else if (s) ++counts[2];
            else ++counts[1];
            continue;
        }
        const int64_t sig = (int64_t)(e == 0 ? f : 128u + f);
        bins[e] += s ? -sig : sig;
        abs_bins[e] += (uint64_t)sig;
    }
    return 0;
}

/*
 * fp8 (NEXT-4): OCP FP8 formats, exact sum as a signed 128-bit integer.
 *   fmt 0 = E4M3 (E4M3FN): s.eeee.mmm, bias 7, no infinities, NaN = s.1111.111;
 *           value = (8+f) * 2^(e-10) for e >= 1, f * 2^-9 for e == 0
 *           -> units of 2^-9: u = (e == 0 ? f : (8+f) << (e-1)).
 *   fmt 1 = E5M2: s.eeeee.mm, bias 15, e == 31: f == 0 -> inf, else NaN;
 *           value = (4+f) * 2^(e-17) for e >= 1, f * 2^-16 for e == 0
 *           -> units of 2^-16: u = (e == 0 ? f : (4+f) << (e-1)).
 * Writes the same record as the binary16 oracle (T, A in those units).
 */
int oracle_exact_sum_fp8(const uint8_t *x, size_t n, int fmt, oracle_sum_result *r) {
    const int ebits = fmt == 0 ? 4 : 5, mbits = fmt == 0 ? 3 : 2;
    const unsigned emax = (1u << ebits) - 1u, mmask = (1u << mbits) - 1u;
    i128 t = 0;
    u128 a = 0;
    uint64_t n_nan = 0, n_pinf = 0, n_ninf = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint8_t h = x[i];
        const unsigned s = (h >> 7) & 1u;
        const unsigned e = (h >> mbits) & emax;
        const unsigned f = h & mmask;
        if (fmt == 0 && e == emax && f == mmask) { ++n_nan; continue; }
        if (fmt == 1 && e == emax) {
            if (f) ++n_nan;
            else if (s) ++n_ninf;
            else ++n_pinf;
            continue;
        }
        const i128 u = e == 0 ? (i128)f : (i128)((1u << mbits) + f) << (e - 1);
        t += s ? -u : u;
        a += (u128)u;
    }
    r->t_lo = (uint64_t)(u128)t;
    r->t_hi = (int64_t)(t >> 64);
    r->a_lo = (uint64_t)a;
    r->a_hi = (uint64_t)(a >> 64);
    r->n_nan = n_nan;
    r->n_pinf = n_pinf;
    r->n_ninf = n_ninf;
    return 0;
}

/*
 * Exact per-segment sums of fp8 inputs (CSR, as oracle_exact_segment_sums_fp16):
 * one oracle_exact_sum_fp8 record per segment.  Returns 0, or -1 if the
 * offsets are decreasing.
 */
int oracle_exact_segment_sums_fp8(const uint8_t *x, const int64_t *offsets, size_t num_segments,
                                  int fmt, oracle_sum_result *r) {
    for (size_t j = 0; j < num_segments; ++j) {
        if (offsets[j + 1] < offsets[j]) return -1;
        oracle_exact_sum_fp8(x + offsets[j], (size_t)(offsets[j + 1] - offsets[j]), fmt, &r[j]);
    }
    return 0;
}
