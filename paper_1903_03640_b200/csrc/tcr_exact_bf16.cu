// tcr_exact_bf16.cu -- NEXT-3 x NEXT-4: bitwise-exact sum of bfloat16 (R(X)
// of Eq. 2, rounded once at the end).
//
// bfloat16 spans 2^-133 .. 2^128, so no single fixed-point word holds every
// input.  Exponents are cut into 8 windows of 32 (k = e >> 5 of the 8-bit
// biased exponent e).  Inside one window every value, placed into a binary64
// as bf16 * 2^-896 (hi word = magnitude bits << 13 | sign, lo word 0: exact
// for normal AND subnormal bf16, the bf16 exponent landing on the binary64
// exponent field), is a multiple of the window's unit and below 2^40 units,
// so up to 2^13 of them add exactly in binary64.
//   fast path  all halves of a warp's iteration lie in one window (or are
//              zero): four binary64 accumulators for that window (no serial
//              DADD chain), flushed every 64 iterations or when the window
//              changes;
//   slow path  mixed windows or inf/NaN in the iteration: each half is turned
//              into an integer of its window's unit and added to a per-lane
//              int64 slot of that window in shared memory.
// Window units (unscaled): u_0 = 2^-133, u_k = 2^(32k - 134) for k >= 1.
// Levels 2-4 add the per-window totals as int128 (order-free); the last CTA
// assembles T = 2 I_0 + sum_k I_k 2^(32k) in units of 2^-134 in a 384-bit
// integer and rounds it once (RNE) to binary32 / binary64.
#include "tcr_bigint.cuh"
#include "tcr_device.cuh"
#include "tcr_int128.cuh"
#include "tcr_internal.h"

namespace tcr {

namespace {

constexpr int kXbWarps = 8;
constexpr int kXbU = 4;
constexpr int kXbAcc = 4;               // independent binary64 accumulators per lane
constexpr int kXbFlushIter = 64;        // 64 iterations x 32 halves = 2^11 adds per lane per flush (<= 2^13 exact)
constexpr int kXbWords = 8 * 2 + 3;     // per CTA partial: 8 x int128 + 3 special counts

// Flushed window accumulator -> integer in the window's unit (exact; < 2^53).
__device__ __forceinline__ long long win_units(double a, int k) {
    // k >= 1: a * 2^(1030 - 32k); k = 0: a * 2^1029 (two exact power-of-two steps)
    const double s2 = k == 0 ? 0x1p514 : ldexp(1.0, 515 - 32 * k);
    return __double2ll_rn((a * 0x1p515) * s2);
}

// One finite nonzero bf16 -> (window, integer in the window's unit).
__device__ __forceinline__ long long half_units(uint32_t h, int& k) {
    const int e = (int)((h >> 7) & 0xFFu);
    const long long m = (long long)(h & 0x7Fu);
    long long v;
    if (e == 0) {
        k = 0;
        v = m;  // subnormal: m * 2^-133
    } else {
        k = e >> 5;
        v = (128 + m) << (k == 0 ? e - 1 : e - 32 * k);
    }
    return (h & 0x8000u) ? -v : v;
}


// RNE binary32 / binary64 of T = 2 I_0 + sum_k I_k 2^(32k) (units 2^-134), or
// the IEEE special value when inf / NaN inputs were counted.
__device__ void finalize_bf16(const i128 (&win)[8], const long long (&c3)[3], float* out_f32,
                              double* out_f64) {
    float f;
    double d;
    if (c3[0] || (c3[1] && c3[2])) {
        f = __int_as_float(0x7FC00000);
        d = __longlong_as_double(0x7FF8000000000000ll);
    } else if (c3[1]) {
        f = __int_as_float(0x7F800000);
        d = __longlong_as_double(0x7FF0000000000000ll);
    } else if (c3[2]) {
        f = __int_as_float(0xFF800000);
        d = __longlong_as_double((long long)0xFFF0000000000000ull);
    } else {
        Big384 B = {{0, 0, 0, 0, 0, 0}};
        big_add_shifted(B, win[0], 1);  // u_0 = 2 * 2^-134
        for (int k = 1; k < 8; ++k) big_add_shifted(B, win[k], 32 * k);
        const bool neg = (long long)B.l[5] < 0;
        if (neg) {  // magnitude: two's complement negate
            unsigned long long carry = 1;
            for (int i = 0; i < 6; ++i) {
                const unsigned long long v = ~B.l[i] + carry;
                carry = (carry && v == 0) ? 1ull : 0ull;
                B.l[i] = v;
            }
        }
        unsigned long long m;
        int e;
        big_round(B, 24, m, e);
        f = ldexpf((float)m, e - 134);  // m <= 2^24 exact; overflow -> inf (IEEE)
        big_round(B, 53, m, e);
        d = ldexp((double)m, e - 134);
        if (neg) {
            f = -f;
            d = -d;
        }
    }
    if (out_f32) *out_f32 = f;
    if (out_f64) *out_f64 = d;
}

__global__ void __launch_bounds__(kXbWarps * 32, 3)
reduce_exact_bf16_kernel(const uint16_t* __restrict__ x, size_t n, long long* out_acc,
                         float* out_f32, double* out_f64, DevWorkspace ws) {
    __shared__ long long s_I[8][kXbWarps * 32];
    pdl_wait_and_release();  // PDL (plain-launch no-op): the previous kernel's writes visible
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) s_I[k][tid] = 0;
    uint32_t cnt[3] = {0u, 0u, 0u};  // NaN, +inf, -inf

    size_t head = ((16u - ((uintptr_t)x & 15u)) & 15u) >> 1;
    if (head > n) head = n;
    const uint16_t* xa = x + head;
    const size_t nb = n - head;
    const size_t T = nb / kTileElems;
    const int tail = (int)(nb - T * kTileElems);
    const size_t W = (size_t)gridDim.x * kXbWarps;
    const size_t w = (size_t)blockIdx.x * kXbWarps + warp;
    const uint4* base = reinterpret_cast<const uint4*>(xa) + lane;

    // kXbAcc independent binary64 accumulators of the current window (the
    // adds of an iteration are spread over them: no serial DADD chain)
    double aw[kXbAcc];
#pragma unroll
    for (int a = 0; a < kXbAcc; ++a) aw[a] = 0.0;
    int wcur = -1;  // window of aw (warp-uniform)
    int it = 0;
    auto flush = [&]() {
        if (wcur >= 0) {
            double t = 0.0;
#pragma unroll
            for (int a = 0; a < kXbAcc; ++a) {
                t += aw[a];  // exact: multiples of the window's unit, total < 2^53 units
                aw[a] = 0.0;
            }
            s_I[wcur][tid] += win_units(t, wcur);
        }
        it = 0;
    };
    auto slow = [&](const uint4& v) {
        const uint32_t ws4[4] = {v.x, v.y, v.z, v.w};
        for (int q = 0; q < 8; ++q) {
            const uint32_t h = (ws4[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
            if ((h & 0x7F80u) == 0x7F80u) {  // inf / NaN
                if (h & 0x7Fu) ++cnt[0];
                else if (h & 0x8000u) ++cnt[2];
                else ++cnt[1];
            } else if (h & 0x7FFFu) {
                int k;
                const long long u = half_units(h, k);
                s_I[k][tid] += u;
            }
        }
    };
    // an iteration's vectors: fast path if every nonzero finite half is in one window.
    // Per word m = the two 15-bit magnitudes; per half t = mag + 0x7FFF as a
    // signed 16-bit value (no carry between halves): zero -> +32767, nonzero
    // -> (mag - 1) - 32768, monotone in mag.  Then the warp's largest
    // magnitude M fixes the window wc = M >> 12 (= biased exponent >> 5), M >=
    // 0x7F80 flags inf / NaN, and "every nonzero half is in window wc" is
    // min over halves of t >= (wc << 12) - 1 - 32768 (zeros pass).  Three
    // SIMD-16x2 operations per word (r02; the r01 test with a per-half zero
    // compare cost ~5 operations per element).
    auto process = [&](const uint4 (&v)[kXbU], int nv) {
        uint32_t vmax = 0u, vmin = 0x7FFF7FFFu;
#pragma unroll
        for (int u = 0; u < kXbU; ++u) {
            if (u >= nv) break;
            const uint32_t ws4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t m = ws4[q] & 0x7FFF7FFFu;
                vmax = __vmaxu2(vmax, m);
                vmin = __vmins2(vmin, m + 0x7FFF7FFFu);
            }
        }
        const uint32_t lmax = max(vmax & 0xFFFFu, vmax >> 16);
        const int lmin = min((int)(short)(vmin & 0xFFFFu), (int)(short)(vmin >> 16));
        const uint32_t M = __reduce_max_sync(0xffffffffu, lmax);
        const uint32_t wc = M >> 12;
        const bool own_ok = lmin >= (int)(wc << 12) - 1 - 32768;
        if (M < 0x7F80u && __all_sync(0xffffffffu, own_ok)) {
            const int k = (int)wc;
            if (k != wcur) {
                flush();
                wcur = k;
            }
#pragma unroll
            for (int u = 0; u < kXbU; ++u) {
                if (u >= nv) break;
                const uint32_t ws4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    // bf16 * 2^-896 as binary64 hi words: sign to bit 31, the
                    // magnitude to bits 13..27 (arithmetic shift keeps the sign)
                    const int hi1 = ((int)ws4[q] >> 3) & (int)0x8FFFE000u;
                    const int hi0 = ((int)(ws4[q] << 16) >> 3) & (int)0x8FFFE000u;
                    aw[(2 * q) % kXbAcc] += __hiloint2double(hi0, 0);
                    aw[(2 * q + 1) % kXbAcc] += __hiloint2double(hi1, 0);
                }
            }
            if (++it == kXbFlushIter) flush();
        } else {
            flush();
            for (int u = 0; u < nv; ++u) slow(v[u]);
        }
    };

    size_t t = w;
    for (; t + (size_t)(kXbU - 1) * W < T; t += (size_t)kXbU * W) {
        uint4 v[kXbU];
#pragma unroll
        for (int u = 0; u < kXbU; ++u) v[u] = ldg_stream(base + (t + (size_t)u * W) * 32);
        __syncwarp();
        process(v, kXbU);
    }
    if (t < T) {  // leftover tiles of this warp: one predicated batch
        uint4 v[kXbU];
#pragma unroll
        for (int u = 0; u < kXbU; ++u)
            v[u] = (t + (size_t)u * W < T) ? ldg_stream(base + (t + (size_t)u * W) * 32)
                                           : make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        process(v, kXbU);
    }
    flush();
    if (w == W - 1) {  // ragged head and tail (zero padded)
        if (head) slow(load_ragged(x, (int)head, lane));
        if (tail) slow(load_ragged(xa + T * kTileElems, tail, lane));
    }
    __syncwarp();

    // levels 2-4: int128 sums per window (order-free) and the special counts
    __shared__ long long s_part[kXbWarps][kXbWords];
    for (int k = 0; k < 8; ++k) {
        const i128 s = warp_sum_i128((i128)s_I[k][tid]);
        if (lane == 0) {
            s_part[warp][2 * k] = (long long)(unsigned long long)s;
            s_part[warp][2 * k + 1] = (long long)(s >> 64);
        }
    }
    for (int c = 0; c < 3; ++c) {
        uint32_t s = cnt[c];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) s_part[warp][16 + c] = s;
    }
    __syncthreads();
    if (warp != 0) return;
    __shared__ unsigned s_last;
    i128 win[8];
    long long c3[3] = {0, 0, 0};
    for (int k = 0; k < 8; ++k) {
        i128 s = 0;
        if (lane < kXbWarps)
            s = (i128)(((u128)(unsigned long long)s_part[lane][2 * k + 1] << 64) |
                       (u128)(unsigned long long)s_part[lane][2 * k]);
        win[k] = warp_sum_i128(s);
    }
    for (int c = 0; c < 3; ++c) {
        long long s = lane < kXbWarps ? s_part[lane][16 + c] : 0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        c3[c] = s;
    }
    if (gridDim.x > 1) {
        long long* parts = reinterpret_cast<long long*>(ws.partials);
        if (lane == 0) {
            long long* p = parts + (size_t)kXbWords * blockIdx.x;
            for (int k = 0; k < 8; ++k) {
                p[2 * k] = (long long)(unsigned long long)win[k];
                p[2 * k + 1] = (long long)(win[k] >> 64);
            }
            for (int c = 0; c < 3; ++c) p[16 + c] = c3[c];
            s_last = (ticket_acq_rel(ws.ticket) == gridDim.x - 1) ? 1u : 0u;
        }
        __syncwarp();  // lane 0's acquire, then the warp's loads below
        if (!__shfl_sync(0xffffffffu, s_last, 0)) return;
        for (int k = 0; k < 8; ++k) {
            i128 s = 0;
            for (int i = lane; i < (int)gridDim.x; i += 32) {
                const long long* p = parts + (size_t)kXbWords * i;
                s += (i128)(((u128)(unsigned long long)__ldcg(p + 2 * k + 1) << 64) |
                            (u128)(unsigned long long)__ldcg(p + 2 * k));
            }
            win[k] = warp_sum_i128(s);
        }
        for (int c = 0; c < 3; ++c) {
            long long s = 0;
            for (int i = lane; i < (int)gridDim.x; i += 32) s += __ldcg(parts + (size_t)kXbWords * i + 16 + c);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            c3[c] = s;
        }
        if (lane == 0) *ws.ticket = 0u;
    }
    if (lane != 0) return;
    if (out_acc) {  // mergeable state: per window 3 limbs of 40/40/48 bits, then the counts
        for (int k = 0; k < 8; ++k) {
            const u128 m = ((u128)1 << 40) - 1;
            out_acc[3 * k] = (long long)((u128)win[k] & m);
            out_acc[3 * k + 1] = (long long)(((u128)win[k] >> 40) & m);
            out_acc[3 * k + 2] = (long long)(win[k] >> 80);
        }
        for (int c = 0; c < 3; ++c) out_acc[24 + c] = c3[c];
    }
    finalize_bf16(win, c3, out_f32, out_f64);
}

__global__ void exact_bf16_finalize_kernel(const long long* acc, float* out_f32, double* out_f64) {
    if (threadIdx.x != 0) return;
    i128 win[8];
    long long c3[3];
    for (int k = 0; k < 8; ++k)
        win[k] = (i128)acc[3 * k] + ((i128)acc[3 * k + 1] << 40) + ((i128)acc[3 * k + 2] << 80);
    for (int c = 0; c < 3; ++c) c3[c] = acc[24 + c];
    finalize_bf16(win, c3, out_f32, out_f64);
}

}  // namespace

cudaError_t launch_reduce_exact_bf16(const uint16_t* x, size_t n, long long* out_acc,
                                     float* out_f32, double* out_f64, const DevWorkspace& ws,
                                     const LaunchCfg& cfg, cudaStream_t stream) {
    const size_t tiles = n / kTileElems;
    size_t g = (tiles + (size_t)kXbWarps * kXbU - 1) / ((size_t)kXbWarps * kXbU);
    size_t gmax = (size_t)cfg.sms * 3;
    const size_t cap = (size_t)ws.capacity / kXbWords;
    if (gmax > cap) gmax = cap;
    if (g > gmax) g = gmax;
    if (g < 1) g = 1;
    launch_maybe_pdl(reduce_exact_bf16_kernel, dim3((unsigned)g), dim3(kXbWarps * 32), 0, stream, cfg.pdl,
                     x, n, out_acc, out_f32, out_f64, ws);
    return cudaGetLastError();
}

cudaError_t launch_exact_bf16_finalize(const long long* acc, float* out_f32, double* out_f64,
                                       cudaStream_t stream) {
    exact_bf16_finalize_kernel<<<1, 32, 0, stream>>>(acc, out_f32, out_f64);
    return cudaGetLastError();
}

}  // namespace tcr
