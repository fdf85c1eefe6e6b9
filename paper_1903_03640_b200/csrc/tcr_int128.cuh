// tcr_int128.cuh -- signed 128-bit integer helpers shared by the kernels that
// sum exactly in units of 2^-24 (every finite binary16 / fp8 value, and every
// fp32 partial the MMA reductions form from them, is an integer multiple of
// 2^-24): warp sums, and the correctly rounded (RNE) conversion of such a sum
// to binary32 / binary64.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tcr {

typedef __int128 i128;
typedef unsigned __int128 u128;

__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int o) {
    const unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
    return (i128)(((u128)hi2 << 64) | (u128)lo2);
}

// Sum over the 32 lanes (all lanes receive it); integer adds: order-free.
__device__ __forceinline__ i128 warp_sum_i128(i128 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += shfl_xor_i128(v, o);
    return v;
}

__device__ __forceinline__ i128 make_i128(long long lo, long long hi) {
    return (i128)(((u128)(unsigned long long)hi << 64) | (u128)(unsigned long long)lo);
}

// Correctly rounded (RNE) value of U * 2^-24 with `bits` significand bits,
// returned as mantissa (<= 2^bits) and binary exponent: value = mant * 2^exp.
__device__ __forceinline__ void round_units(u128 U, int bits, unsigned long long& mant, int& exp) {
    if (U == 0) {
        mant = 0;
        exp = 0;
        return;
    }
    const unsigned long long hi = (unsigned long long)(U >> 64), lo = (unsigned long long)U;
    const int msb = hi ? 127 - __clzll((long long)hi) : 63 - __clzll((long long)lo);
    if (msb < bits) {  // exact
        mant = lo;
        exp = -24;
        return;
    }
    const int shift = msb - (bits - 1);
    u128 q = U >> shift;
    const u128 rem = U - (q << shift);
    const u128 halfway = (u128)1 << (shift - 1);
    if (rem > halfway || (rem == halfway && (q & 1))) ++q;
    mant = (unsigned long long)q;  // may equal 2^bits after rounding up: still exact below
    exp = shift - 24;
}

// RNE binary32 and binary64 of T * 2^-24 (|T| < 2^127; no overflow below 2^104).
__device__ __forceinline__ void round_units_f32_f64(i128 T, float& f, double& d) {
    const bool neg = T < 0;
    const u128 U = neg ? (u128)(-T) : (u128)T;
    unsigned long long m;
    int e;
    round_units(U, 24, m, e);
    f = ldexpf((float)m, e);  // m <= 2^24: exact; the scaling is exact
    round_units(U, 53, m, e);
    d = ldexp((double)m, e);
    if (neg) {
        f = -f;
        d = -d;
    }
}

}  // namespace tcr
