// tcr_bigint.cuh -- a 384-bit two's complement integer for the exact
// bfloat16 reduction (its sums span more than 128 bits): add an int128 at a
// bit offset, and round the magnitude once (RNE) to a given number of
// significant bits.
#pragma once

#include "tcr_int128.cuh"

namespace tcr {

// 384-bit two's complement accumulator: limbs l[0] (least significant) .. l[5].
struct Big384 {
    unsigned long long l[6];
};

__device__ __forceinline__ void big_add_shifted(Big384& B, i128 v, int shift) {  // B += v * 2^shift (mod 2^384)
    const unsigned long long ext = v < 0 ? ~0ull : 0ull;
    unsigned long long e[7];  // v sign-extended to 448 bits
    e[0] = (unsigned long long)v;
    e[1] = (unsigned long long)(v >> 64);
    for (int i = 2; i < 7; ++i) e[i] = ext;
    const int q = shift >> 6, r = shift & 63;
    unsigned long long carry = 0;
    for (int i = 0; i < 6; ++i) {
        const int j = i - q;
        unsigned long long w = 0;
        if (j >= 0) w = r ? (e[j] << r) : e[j];
        if (r && j - 1 >= 0) w |= e[j - 1] >> (64 - r);
        const unsigned long long a0 = B.l[i];
        const unsigned long long s1 = a0 + w;
        const unsigned long long c1 = s1 < a0 ? 1ull : 0ull;
        const unsigned long long s2 = s1 + carry;
        const unsigned long long c2 = s2 < s1 ? 1ull : 0ull;
        B.l[i] = s2;
        carry = c1 | c2;
    }
}

// RNE of the non-negative 384-bit M (units 2^-134) to `bits` significant bits:
// value = mant * 2^(exp - 134).
__device__ __forceinline__ void big_round(const Big384& M, int bits, unsigned long long& mant, int& exp) {
    int top = -1;
    for (int i = 5; i >= 0 && top < 0; --i)
        if (M.l[i]) top = i * 64 + 63 - __clzll((long long)M.l[i]);
    if (top < 0) {
        mant = 0;
        exp = 0;
        return;
    }
    auto bit = [&](int p) -> unsigned long long { return (M.l[p >> 6] >> (p & 63)) & 1ull; };
    if (top < bits) {  // fits: exact
        unsigned long long m = 0;
        for (int p = top; p >= 0; --p) m = (m << 1) | bit(p);
        mant = m;
        exp = 0;
        return;
    }
    const int shift = top - (bits - 1);
    unsigned long long q = 0;
    for (int p = top; p >= shift; --p) q = (q << 1) | bit(p);
    const unsigned long long half = bit(shift - 1);
    bool sticky = false;
    for (int p = shift - 2; p >= 0 && !sticky; --p) sticky = bit(p) != 0;
    if (half && (sticky || (q & 1ull))) ++q;  // may reach 2^bits: still exact below
    mant = q;
    exp = shift;
}

// Two's complement negate (magnitude of a negative value).
__device__ __forceinline__ void big_negate(Big384& B) {
    unsigned long long carry = 1;
    for (int i = 0; i < 6; ++i) {
        const unsigned long long v = ~B.l[i] + carry;
        carry = (carry && v == 0) ? 1ull : 0ull;
        B.l[i] = v;
    }
}

}  // namespace tcr
