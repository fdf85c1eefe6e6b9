// tcr_exact.cu -- NEXT-3: bitwise-exact sum of binary16 (R(X) of Eq. 2,
// P:106-110, with no rounding at all until the final conversion).
//
// Every finite binary16 value is an integer multiple of 2^-24 below 2^16.
// Placing its 15 magnitude bits at bit 42 of a binary64 (and its sign at
// bit 63) gives a binary64 equal to the value times 2^-1008 -- exact for
// normal AND subnormal inputs (the subnormal binary16 f*2^-24 lands on the
// binary64 subnormal f*2^-1032).  All such numbers are multiples of 2^-1032,
// so binary64 additions of up to 8192 of them (|sum| < 2^-979, i.e. fewer
// than 53 significant bits) are exact.  Each lane therefore adds scaled
// binary64 values in two or four accumulators, flushes them every kFlushIter
// iterations (<= 1024 elements per accumulator) into a signed 128-bit
// integer in units of 2^-24, and the warp / CTA / grid levels add int128
// exactly (the same last-CTA completion as the MMA kernels).  The result is
// independent of thread count and order: it equals the exact integer
// T = sum x_i * 2^24 of Eq. 2 bit for bit, and the binary32 / binary64 outputs are the correctly
// rounded (RNE) values of T * 2^-24.
//
// Accumulator state for sharded use: int64 acc[6] = {l0, l1, l2, n_nan,
// n_pinf, n_ninf} with T = l0 + l1*2^40 + l2*2^80 (l0, l1 in [0, 2^40)); an
// integer SUM-allreduce of acc[] over GPUs is exact, and
// tcr_exact_finalize() rounds it.
#include "tcr_device.cuh"
#include "tcr_int128.cuh"
#include "tcr_internal.h"
#include "tcr_peer.cuh"
#include "tcr_sm100.cuh"

#include <map>
#include <mutex>

namespace tcr {

namespace {

constexpr int kExactWarps = 8;
constexpr int kExactUnroll = 4;
constexpr int kFlushIter = 64;  // 64 iterations x 4 vectors x 4 halves = 1024 per accumulator

// Scaled binary64 of the low / high binary16 of a 32-bit word (x 2^-1008):
// the high 32 bits of the binary64 are sign | 0000 | e(5) | f(10) | 0...,
// i.e. the binary16 arithmetic-shifted right by 6 (from bit 31) with the
// sign copies in bits 25..30 masked off.  Low 32 bits are zero.
__device__ __forceinline__ double scaled_lo(uint32_t w) {
    const uint32_t hi = (uint32_t)((int)(w << 16) >> 6) & 0x81FFFC00u;
    return __hiloint2double((int)hi, 0);
}
__device__ __forceinline__ double scaled_hi(uint32_t w) {
    const uint32_t hi = (uint32_t)((int)w >> 6) & 0x81FFFC00u;
    return __hiloint2double((int)hi, 0);
}

// Non-finite detection: x * 0 is NaN exactly when x is inf or NaN, so one
// HFMA2 per 32-bit word folds the test into a half2 "probe" that stays +-0
// unless a special value went by; it is checked once per iteration.
__device__ __forceinline__ uint32_t probe_word(uint32_t w, uint32_t probe) {
    const __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&w), __float2half2_rn(0.0f),
                              *reinterpret_cast<const __half2*>(&probe));
    return *reinterpret_cast<const uint32_t*>(&r);
}

// Rare path: count the non-finite halves of v and subtract the scaled
// binary64 values they contributed (exactly: every partial sum stays a
// multiple of 2^-1032 below 2^-979).
template <int NA>
__device__ __forceinline__ void fix_specials(const uint4& v, double (&a)[NA], uint32_t (&cnt)[3]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    for (int k = 0; k < 4; ++k) {
        for (int h = 0; h < 2; ++h) {
            const uint32_t half = (w[k] >> (16 * h)) & 0xFFFFu;
            if ((half & 0x7C00u) == 0x7C00u) {
                if (half & 0x3FFu) ++cnt[0];            // NaN
                else if (half & 0x8000u) ++cnt[2];      // -inf
                else ++cnt[1];                          // +inf
                // the accumulator exact_vec added it to: word parity, half
                if (h == 0) a[(2 * (k & 1)) % NA] -= scaled_lo(w[k]);
                else a[(2 * (k & 1) + 1) % NA] -= scaled_hi(w[k]);
            }
        }
    }
}

// NA accumulators (2 or 4): word k's low / high half go to a[(2(k&1)) % NA]
// / a[(2(k&1)+1) % NA]; with NA = 4 an iteration's adds form four independent
// DADD chains (r02: two chains left the binary16 kernel FP64-latency-bound).
template <int NA>
__device__ __forceinline__ void exact_vec(const uint4& v, double (&a)[NA], uint32_t& probe) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        probe = probe_word(w[k], probe);
        a[(2 * (k & 1)) % NA] += scaled_lo(w[k]);
        a[(2 * (k & 1) + 1) % NA] += scaled_hi(w[k]);
    }
}

// fp8 (E4M3 / E5M2) -> binary16 is exact (every fp8 value is a binary16
// value; cvt.rn.f16x2.{e4m3,e5m2}x2): 16 fp8 bytes become two vectors of 8
// binary16 that go through the same exact accumulation (NEXT-3 x NEXT-4).
// One loaded 16-byte vector of format F into the accumulators.
template <int F, int NA>
__device__ __forceinline__ void exact_vec_f(const uint4& v, double (&a)[NA], uint32_t& probe) {
    if constexpr (F == kF16) {
        exact_vec<NA>(v, a, probe);
    } else {  // word by word: two binary16 pairs per 32-bit word, few live registers
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint16_t b = (uint16_t)(w[k] >> (16 * h));
                uint32_t o;
                if constexpr (F == kE4M3) asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(o) : "h"(b));
                else asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(o) : "h"(b));
                // converted word j = 2k + h: parity of j (= h) picks the pair,
                // as fix_specials_f's word index in lo / hi does
                probe = probe_word(o, probe);
                a[(2 * h) % NA] += scaled_lo(o);
                a[(2 * h + 1) % NA] += scaled_hi(o);
            }
        }
    }
}

template <int F, int NA>
__device__ __forceinline__ void fix_specials_f(const uint4& v, double (&a)[NA], uint32_t (&cnt)[3]) {
    if constexpr (F == kF16) {
        fix_specials<NA>(v, a, cnt);
    } else {  // word by word, as exact_vec_f converts (few live registers)
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            const uint16_t b = (uint16_t)(w[j >> 1] >> (16 * (j & 1)));
            uint32_t o;
            if constexpr (F == kE4M3) asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(o) : "h"(b));
            else asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(o) : "h"(b));
            for (int h = 0; h < 2; ++h) {
                const uint32_t half = (o >> (16 * h)) & 0xFFFFu;
                if ((half & 0x7C00u) == 0x7C00u) {
                    if (half & 0x3FFu) ++cnt[0];
                    else if (half & 0x8000u) ++cnt[2];
                    else ++cnt[1];
                    // converted word j went to the pair of parity j & 1
                    if (h == 0) a[(2 * (j & 1)) % NA] -= scaled_lo(o);
                    else a[(2 * (j & 1) + 1) % NA] -= scaled_hi(o);
                }
            }
        }
    }
}

// Exact conversion of a flushed accumulator to integer units of 2^-24.
__device__ __forceinline__ long long to_units(double a) {
    return __double2ll_rn((a * 0x1p1008) * 0x1p24);  // both scalings exact; result < 2^53
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Split an int128 into limbs l0 + l1*2^40 + l2*2^80 (l0, l1 in [0, 2^40)).
__device__ __forceinline__ void to_limbs(i128 t, long long* acc) {
    const u128 m = ((u128)1 << 40) - 1;
    acc[0] = (long long)((u128)t & m);
    acc[1] = (long long)(((u128)t >> 40) & m);
    acc[2] = (long long)(t >> 80);
}

__device__ __forceinline__ i128 from_limbs(const long long* acc) {
    return (i128)acc[0] + ((i128)acc[1] << 40) + ((i128)acc[2] << 80);
}

__device__ void finalize(const long long* acc, float* out_f32, double* out_f64) {
    float f;
    double d;
    const long long n_nan = acc[3], n_pinf = acc[4], n_ninf = acc[5];
    if (n_nan || (n_pinf && n_ninf)) {
        f = __int_as_float(0x7FC00000);
        d = __longlong_as_double(0x7FF8000000000000ll);
    } else if (n_pinf) {
        f = __int_as_float(0x7F800000);
        d = __longlong_as_double(0x7FF0000000000000ll);
    } else if (n_ninf) {
        f = __int_as_float(0xFF800000);
        d = __longlong_as_double((long long)0xFFF0000000000000ull);
    } else {
        const i128 T = from_limbs(acc);
        const bool neg = T < 0;
        const u128 U = neg ? (u128)(-T) : (u128)T;
        unsigned long long m;
        int e;
        round_units(U, 24, m, e);
        f = ldexpf((float)m, e);  // m <= 2^24: exact; scaling by 2^e exact (no overflow below 2^104)
        round_units(U, 53, m, e);
        d = ldexp((double)m, e);
        if (neg) {
            f = -f;
            d = -d;
        }
    }
    if (out_f32) *out_f32 = f;
    if (out_f64) *out_f64 = d;
}

// Levels 2-4 of the exact kernels: warp, CTA and grid as exact integer adds
// (order-free), then the fused peer combine of the limbs (kPeer) or the
// final rounding.  Every thread calls it with its lane's int128 and special
// counts; WARPS warps per CTA; chunk_next (if not null) is reset by the last
// CTA (the bulk kernel's dynamic tail).
template <int WARPS, bool kPeer>
__device__ __forceinline__ void exact_complete(i128 acc, uint32_t (&cnt)[3], long long* out_acc,
                                               float* out_f32, double* out_f64, const DevWorkspace& ws,
                                               const PeerCombine& pc, int me, unsigned* chunk_next) {
    constexpr int kExactWarps = WARPS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp, CTA and grid levels: exact integer adds (order-free)
    __shared__ long long s_part[kExactWarps][5];
    __shared__ unsigned s_last;
    acc = warp_sum_i128(acc);
    for (int k = 0; k < 3; ++k) cnt[k] = warp_sum_u32(cnt[k]);
    if (lane == 0) {
        s_part[warp][0] = (long long)(unsigned long long)acc;
        s_part[warp][1] = (long long)(acc >> 64);
        for (int k = 0; k < 3; ++k) s_part[warp][2 + k] = cnt[k];
    }
    __syncthreads();
    if (warp != 0) return;
    const unsigned long long prev = kPeer ? peer_counter(pc, me) : 0ull;
    i128 b = 0;
    long long c[3] = {0, 0, 0};
    if (lane < kExactWarps) {
        b = (i128)(((u128)(unsigned long long)s_part[lane][1] << 64) |
                   (u128)(unsigned long long)s_part[lane][0]);
        for (int k = 0; k < 3; ++k) c[k] = s_part[lane][2 + k];
    }
    b = warp_sum_i128(b);
    for (int k = 0; k < 3; ++k)
        for (int o = 16; o > 0; o >>= 1) c[k] += __shfl_xor_sync(0xffffffffu, c[k], o);
    long long res[6];
    if (gridDim.x > 1) {
        // CTA partial: 5 int64 words per CTA in the workspace (reinterpreted doubles)
        long long* parts = reinterpret_cast<long long*>(ws.partials);
        if (lane == 0) {
            long long* p = parts + 5 * (size_t)blockIdx.x;
            p[0] = (long long)(unsigned long long)b;
            p[1] = (long long)(b >> 64);
            p[2] = c[0];
            p[3] = c[1];
            p[4] = c[2];
            if constexpr (kPeer) {  // fence + relaxed ticket: no spill in the peer variant
                __threadfence();
                s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
            } else {
                s_last = (ticket_acq_rel(ws.ticket) == gridDim.x - 1) ? 1u : 0u;
            }
        }
        __syncwarp();  // lane 0's acquire, then the warp's loads below
        if (!__shfl_sync(0xffffffffu, s_last, 0)) return;
        if constexpr (kPeer) __threadfence();
        b = 0;
        c[0] = c[1] = c[2] = 0;
        for (int i = lane; i < (int)gridDim.x; i += 32) {
            const long long* p = parts + 5 * (size_t)i;
            b += (i128)(((u128)(unsigned long long)__ldcg(p + 1) << 64) |
                        (u128)(unsigned long long)__ldcg(p));
            c[0] += __ldcg(p + 2);
            c[1] += __ldcg(p + 3);
            c[2] += __ldcg(p + 4);
        }
        b = warp_sum_i128(b);
        for (int k = 0; k < 3; ++k)
            for (int o = 16; o > 0; o >>= 1) c[k] += __shfl_xor_sync(0xffffffffu, c[k], o);
        if (lane == 0) {
            *ws.ticket = 0u;
            if (chunk_next) *chunk_next = 0u;
        }
    } else if (lane == 0 && chunk_next) {
        *chunk_next = 0u;
    }
    if constexpr (kPeer) {
        // every lane computes the limbs (b, c are warp-uniform after the sums)
        to_limbs(b, res);
        res[3] = c[0];
        res[4] = c[1];
        res[5] = c[2];
        const bool ok = peer_combine_exact(res, pc, me, lane, prev);
        if (lane == 0) {
            if (out_acc)
                for (int k = 0; k < 6; ++k) out_acc[k] = res[k];
            if (ok) {
                finalize(res, out_f32, out_f64);
            } else {
                if (out_f32) *out_f32 = __int_as_float(0x7FC00000);
                if (out_f64) *out_f64 = __longlong_as_double(0x7FF8000000000000ll);
            }
        }
        return;
    }
    if (lane == 0) {
        to_limbs(b, res);
        res[3] = c[0];
        res[4] = c[1];
        res[5] = c[2];
        if (out_acc)
            for (int k = 0; k < 6; ++k) out_acc[k] = res[k];
        finalize(res, out_f32, out_f64);
    }
}

// kPeer: the NEXT-2 x NEXT-3 variant -- the last CTA combines the limbs
// with the peers' over NVLink mailboxes (tcr_peer.cuh); grid.y slices =
// emulated ranks, as in reduce_stream_kernel.
template <int U, bool kPeer, int F = kF16>
__global__ void __launch_bounds__(kExactWarps * 32, (U <= 4 ? 4 : 3))
reduce_exact_kernel(const uint8_t* __restrict__ x, size_t n, long long* out_acc, float* out_f32,
                    double* out_f64, DevWorkspace ws, PeerCombine pc) {
    constexpr int ES = FmtInfo<F>::kBytes;
    constexpr int kTileBytes = 512;
    // PDL (plain-launch no-op): the previous kernel's writes visible.  The
    // peer variant always launches plainly (it waits on other ranks).
    if constexpr (!kPeer) pdl_wait_and_release();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int me = pc.rank;
    if (kPeer && gridDim.y > 1) {  // emulated peer group: slice y is rank y
        const size_t P = gridDim.y, r = blockIdx.y;
        const size_t lo = r * n / P, hi = (r + 1) * n / P;
        x += lo * ES;
        n = hi - lo;
        ws.partials += 5 * r * gridDim.x;  // 5 int64 words per CTA (stored in the doubles)
        ws.ticket += r;
        if (out_acc) out_acc += 6 * r;
        if (out_f32) out_f32 += r;
        if (out_f64) out_f64 += r;
        me = (int)r;
    }
    const size_t nbytes = n * ES;
    size_t head = (16u - ((uintptr_t)x & 15u)) & 15u;  // bytes before the first 16-B boundary
    if (head > nbytes) head = nbytes;
    const uint8_t* xa = x + head;
    const size_t nb = nbytes - head;
    const size_t T = nb / kTileBytes;
    const int tail = (int)(nb - T * kTileBytes);
    const size_t W = (size_t)gridDim.x * kExactWarps;
    const size_t w = (size_t)blockIdx.x * kExactWarps + warp;
    const uint4* base = reinterpret_cast<const uint4*>(xa) + lane;
    // <= 1024 binary16 per accumulator between flushes (an fp8 vector is 16 of them)
    constexpr int kFlush = kFlushIter * kExactUnroll / U / (ES == 1 ? 2 : 1);

    // four accumulators at U = 8 (the default); two at U = 4, where 4 CTAs/SM
    // leave 64 registers
    constexpr int NA = U >= 8 ? 4 : 2;
    i128 acc = 0;
    double a[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) a[i] = 0.0;
    auto drain = [&]() {
#pragma unroll
        for (int i = 0; i < NA; ++i) {
            acc += (i128)to_units(a[i]);
            a[i] = 0.0;
        }
    };
    uint32_t cnt[3] = {0u, 0u, 0u};
    uint32_t probe = 0u;
    int it = 0;
    size_t t = w;
    for (; t + (size_t)(U - 1) * W < T; t += (size_t)U * W) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream(base + (t + (size_t)u * W) * 32);
        __syncwarp();  // scheduling fence: all U loads issue before the first consumer
#pragma unroll
        for (int u = 0; u < U; ++u) exact_vec_f<F, NA>(v[u], a, probe);
        if (probe & 0x7FFF7FFFu) {  // some half was inf or NaN (rare): reload and fix
#pragma unroll 1
            for (int u = 0; u < U; ++u)
                fix_specials_f<F, NA>(ldg_stream(base + (t + (size_t)u * W) * 32), a, cnt);
            probe = 0u;
        }
        if (++it == kFlush) {
            it = 0;
            drain();
        }
    }
    auto one = [&](const uint4& v) {
        uint32_t p = 0u;
        exact_vec_f<F, NA>(v, a, p);
        if (p & 0x7FFF7FFFu) fix_specials_f<F, NA>(v, a, cnt);
    };
    if (t < T) {  // fewer than U tiles left for this warp: one predicated batch (one latency)
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            v[u] = (t + (size_t)u * W < T) ? ldg_stream(base + (t + (size_t)u * W) * 32)
                                           : make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) one(v[u]);
    }
    if (w == W - 1) {  // ragged head and tail
        if (head) one(load_ragged_bytes(x, (int)head, lane));
        if (tail) one(load_ragged_bytes(xa + T * kTileBytes, tail, lane));
    }
    drain();

    exact_complete<kExactWarps, kPeer>(acc, cnt, out_acc, out_f32, out_f64, ws, pc, me, nullptr);
}

// TMA-fed exact reduction with a dynamic tail (r02 §18; binary16 / fp8, the
// default exact kernel from 512 MiB): a producer lane streams 32 KiB chunks
// into a 4-stage SMEM ring with cp.async.bulk -- CTA b its contiguous run of
// the first 92 % of the chunks, then chunks by ticket (ws.chunk_next, two
// tickets held ahead) -- and 8 consumer warps apply the same exact per-vector
// accumulation as reduce_exact_kernel to the stage (warp w: 512-byte tiles w,
// w + 8, ...).  Integer levels 2-4 are order-free, so which CTA took which
// chunk cannot change a bit.  Bytes in flight are bounded by SMEM (128 KiB
// per SM), not by registers, and the tail does not wait for the slowest SM.
constexpr int kXbConsumers = 8;
constexpr int kXbThreads = (kXbConsumers + 1) * 32;
constexpr uint32_t kXbStageBytes = 32768;
constexpr uint32_t kXbHeader = 1024;

__device__ __forceinline__ uint4 lds128x(const void* p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(sm100::smem_addr(p)));
    return r;
}

// kPeer: the NEXT-2 x NEXT-3 variant (the limb combine with the peers fused
// into the last CTA); grid.y slices = emulated ranks, as reduce_exact_kernel.
template <int F, bool kPeer = false>
__global__ void __launch_bounds__(kXbThreads, 1)
reduce_exact_bulk_kernel(const uint8_t* __restrict__ x, size_t n, int stages, int dyn_pct,
                         long long* out_acc, float* out_f32, double* out_f64, DevWorkspace ws,
                         PeerCombine pc) {
    constexpr int ES = FmtInfo<F>::kBytes;
    constexpr int kTileBytes = 512;
    constexpr int NA = 4;
    constexpr int kTilesPerWarp = (int)(kXbStageBytes / kTileBytes) / kXbConsumers;  // 8 per stage
    // <= 1024 binary16 per accumulator between flushes: a tile gives each of
    // the 4 accumulators 2 (binary16) or 4 (fp8 as binary16) values per lane
    constexpr int kFlushStages = (ES == 1 ? 256 : 512) / (2 * kTilesPerWarp);
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + stages;
    volatile uint32_t* sinfo = reinterpret_cast<volatile uint32_t*>(empty + stages);  // [stages]
    uint8_t* ring = smem + kXbHeader;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int me = pc.rank;
    if (kPeer && gridDim.y > 1) {  // emulated peer group: slice y is rank y, reducing its shard
        const size_t P = gridDim.y, r = blockIdx.y;
        const size_t lo = r * n / P, hi = (r + 1) * n / P;
        x += lo * ES;
        n = hi - lo;
        ws.partials += 5 * r * gridDim.x;  // 5 int64 words per CTA
        ws.ticket += r;
        ws.chunk_next += r;
        if (out_acc) out_acc += 6 * r;
        if (out_f32) out_f32 += r;
        if (out_f64) out_f64 += r;
        me = (int)r;
    }

    const size_t nbytes = n * ES;
    size_t head = (16u - ((uintptr_t)x & 15u)) & 15u;
    if (head > nbytes) head = nbytes;
    const uint8_t* xa = x + head;
    const size_t nb = nbytes - head;
    const size_t C = nb / kXbStageBytes;
    const size_t D = C * (size_t)dyn_pct / 100u;
    const size_t Cs = C - D;
    const size_t G = gridDim.x, b = blockIdx.x;
    const size_t c_begin = b * Cs / G;
    const long long nstatic = (long long)((b + 1) * Cs / G - c_begin);

    if (threadIdx.x == 0) {
        for (int st = 0; st < stages; ++st) {
            sm100::mbar_init(&full[st], 1);
            sm100::mbar_init(&empty[st], kXbConsumers);
        }
        sm100::fence_mbar_init();
    }
    __syncthreads();
    if constexpr (!kPeer) pdl_wait_and_release();  // PDL: no global memory before the previous kernel completes

    i128 acc = 0;
    uint32_t cnt[3] = {0u, 0u, 0u};
    if (warp == kXbConsumers) {  // producer lane: static run, tickets, END
        if (lane == 0) {
            const uint64_t pol = sm100::policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            auto issue = [&](size_t c) {
                sm100::mbar_wait(&empty[st], ph ^ 1u);
                sinfo[st] = 1u;
                sm100::mbar_arrive_expect_tx(&full[st], kXbStageBytes);
                sm100::bulk_g2s(ring + (size_t)st * kXbStageBytes, xa + c * (size_t)kXbStageBytes,
                                kXbStageBytes, &full[st], pol);
                if (++st == stages) {
                    st = 0;
                    ph ^= 1u;
                }
            };
            unsigned t0 = 0u, t1 = 0u;
            bool f0 = false, f1 = false;
            for (long long i = 0; i < nstatic; ++i) {
                if (D && !f0 && nstatic - i <= 2) {
                    t0 = atomicAdd(ws.chunk_next, 1u);
                    f0 = true;
                }
                if (D && !f1 && nstatic - i <= 1) {
                    t1 = atomicAdd(ws.chunk_next, 1u);
                    f1 = true;
                }
                issue(c_begin + (size_t)i);
            }
            if (D) {
                if (!f0) t0 = atomicAdd(ws.chunk_next, 1u);
                if (!f1) t1 = atomicAdd(ws.chunk_next, 1u);
                for (;;) {
                    const unsigned t = t0;
                    t0 = t1;
                    t1 = atomicAdd(ws.chunk_next, 1u);
                    if ((size_t)t >= D) break;
                    issue(Cs + (size_t)t);
                }
            }
            sm100::mbar_wait(&empty[st], ph ^ 1u);  // END: a stage with no bytes
            sinfo[st] = 0u;
            sm100::mbar_arrive(&full[st]);
        }
        __syncwarp();
    } else {  // consumer warps
        double a[NA];
#pragma unroll
        for (int i = 0; i < NA; ++i) a[i] = 0.0;
        auto drain = [&]() {
#pragma unroll
            for (int i = 0; i < NA; ++i) {
                acc += (i128)to_units(a[i]);
                a[i] = 0.0;
            }
        };
        int st = 0, it = 0;
        uint32_t ph = 0;
        for (;;) {
            sm100::mbar_wait(&full[st], ph);
            if (sinfo[st] == 0u) break;
            const uint8_t* stage = ring + (size_t)st * kXbStageBytes + lane * 16;
            uint4 v[kTilesPerWarp];
#pragma unroll
            for (int k = 0; k < kTilesPerWarp; ++k) v[k] = lds128x(stage + (size_t)(warp + k * kXbConsumers) * kTileBytes);
            uint32_t probe = 0u;
#pragma unroll
            for (int k = 0; k < kTilesPerWarp; ++k) exact_vec_f<F, NA>(v[k], a, probe);
            if (probe & 0x7FFF7FFFu) {  // some half was inf or NaN (rare): fix from SMEM
#pragma unroll 1
                for (int k = 0; k < kTilesPerWarp; ++k)
                    fix_specials_f<F, NA>(lds128x(stage + (size_t)(warp + k * kXbConsumers) * kTileBytes), a, cnt);
            }
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&empty[st]);  // stage consumed by this warp
            if (++it == kFlushStages) {
                it = 0;
                drain();
            }
            if (++st == stages) {
                st = 0;
                ph ^= 1u;
            }
        }
        auto one = [&](const uint4& v) {
            uint32_t p = 0u;
            exact_vec_f<F, NA>(v, a, p);
            if (p & 0x7FFF7FFFu) fix_specials_f<F, NA>(v, a, cnt);
        };
        if (blockIdx.x == gridDim.x - 1) {  // ragged work past the last chunk, and the head
            const uint8_t* xr = xa + C * (size_t)kXbStageBytes;
            const size_t rem = nb - C * (size_t)kXbStageBytes;
            const size_t Tr = rem / kTileBytes;
            const int tail = (int)(rem - Tr * kTileBytes);
            const uint4* base = reinterpret_cast<const uint4*>(xr) + lane;
            drain();
            int k = 0;
            for (size_t t = warp; t < Tr; t += kXbConsumers) {
                one(ldg_stream(base + t * 32));
                if (++k == 32) {  // <= 1024 values per accumulator between flushes
                    k = 0;
                    drain();
                }
            }
            if (warp == 0 && head) one(load_ragged_bytes(x, (int)head, lane));
            if (warp == 1 && tail) one(load_ragged_bytes(xr + Tr * kTileBytes, tail, lane));
        }
        drain();
    }
    exact_complete<kXbConsumers + 1, kPeer>(acc, cnt, out_acc, out_f32, out_f64, ws, pc, me,
                                            D ? ws.chunk_next : nullptr);
}

__global__ void exact_finalize_kernel(const long long* acc, float* out_f32, double* out_f64) {
    if (threadIdx.x == 0) {
        long long a[6];
        for (int k = 0; k < 6; ++k) a[k] = acc[k];
        finalize(a, out_f32, out_f64);
    }
}

}  // namespace

int exact_grid(size_t n, const LaunchCfg& cfg, int capacity_words) {
    const size_t tiles = n / kTileElems;
    const size_t per_cta = (size_t)kExactWarps * kExactUnroll;
    size_t g = (tiles + per_cta - 1) / per_cta;
    size_t gmax = (size_t)cfg.sms * (cfg.exact_bps < 1 ? 4 : cfg.exact_bps);
    const size_t cap = (size_t)capacity_words / 5;  // 5 int64 words per CTA partial
    if (gmax > cap) gmax = cap;
    if (g > gmax) g = gmax;
    return g < 1 ? 1 : (int)g;
}

template <int F>
static cudaError_t launch_exact_bulk(const uint8_t* x, size_t n, long long* out_acc, float* out_f32,
                                     double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                     cudaStream_t stream) {
    constexpr int kStages = 4;
    const size_t smem = kXbHeader + (size_t)kStages * kXbStageBytes;
    auto kernel = reduce_exact_bulk_kernel<F>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        static std::mutex mu;
        static std::map<int, size_t> configured;
        std::lock_guard<std::mutex> lk(mu);
        if (smem > configured[dev]) {
            if ((e = cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem)))
                return e;
            configured[dev] = smem;
        }
    }
    const size_t C = n * FmtInfo<F>::kBytes / kXbStageBytes;
    size_t g = (size_t)cfg.sms;
    if (g > C) g = C;
    if (g < 1) g = 1;
    // the dynamic tail when every CTA streams >= TCR_CFG_TC05_DYN_MIN_RUN chunks
    const int dyn = (C >= (size_t)cfg.tc05_dyn_min_run * g) ? cfg.tc05_dynamic : 0;
    const PeerCombine none{};
    launch_maybe_pdl(kernel, dim3((unsigned)g), dim3(kXbThreads), smem, stream, cfg.pdl, x, n, kStages, dyn,
                     out_acc, out_f32, out_f64, ws, none);
    return cudaGetLastError();
}

template <int F>
static cudaError_t launch_exact_f(const uint8_t* x, size_t n, long long* out_acc, float* out_f32,
                                  double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                  cudaStream_t stream) {
    // binary16: TMA-fed with the dynamic tail from 128 MiB (r02 §18: 0.90-0.94 x
    // the LDG kernel's time from 2^26 to 2^32); fp8, ALU-bound by its
    // conversions, keeps the LDG kernel's 24 warps per SM (1.05 x at 2^31 on
    // 8 consumer warps, profiles/r02/exact_bulk_ab2.txt)
    if (cfg.exact_bulk == 2 ||
        (cfg.exact_bulk == 1 && F == kF16 && n * FmtInfo<F>::kBytes >= ((size_t)128 << 20)))
        return launch_exact_bulk<F>(x, n, out_acc, out_f32, out_f64, ws, cfg, stream);
    // grid from the input bytes (in 2-byte element equivalents)
    const int g = exact_grid(n * FmtInfo<F>::kBytes / 2, cfg, ws.capacity);
    const PeerCombine none{};
    if (cfg.exact_unroll == 8)
        launch_maybe_pdl(reduce_exact_kernel<8, false, F>, dim3(g), dim3(kExactWarps * 32), 0, stream,
                         cfg.pdl, x, n, out_acc, out_f32, out_f64, ws, none);
    else
        launch_maybe_pdl(reduce_exact_kernel<4, false, F>, dim3(g), dim3(kExactWarps * 32), 0, stream,
                         cfg.pdl, x, n, out_acc, out_f32, out_f64, ws, none);
    return cudaGetLastError();
}

cudaError_t launch_reduce_exact(int fmt, const void* x, size_t n, long long* out_acc,
                                float* out_f32, double* out_f64, const DevWorkspace& ws,
                                const LaunchCfg& cfg, cudaStream_t stream) {
    const uint8_t* xb = static_cast<const uint8_t*>(x);
    switch (fmt) {
        case kE4M3: return launch_exact_f<kE4M3>(xb, n, out_acc, out_f32, out_f64, ws, cfg, stream);
        case kE5M2: return launch_exact_f<kE5M2>(xb, n, out_acc, out_f32, out_f64, ws, cfg, stream);
        case kF16: return launch_exact_f<kF16>(xb, n, out_acc, out_f32, out_f64, ws, cfg, stream);
        default: return cudaErrorInvalidValue;  // bfloat16 has its own kernel (tcr_exact_bf16.cu)
    }
}

// The TMA-fed exact kernel fused with the peer limb combine (binary16): a
// plain launch per real rank; emulated ranks in one cooperative launch
// (grid.y = ranks; one CTA per SM, so at most SMs / P CTAs per rank).
static cudaError_t launch_exact_bulk_peer(const uint8_t* x, size_t n, long long* out_acc, float* out_f32,
                                          double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                          const PeerCombine& pc, bool emulate, cudaStream_t stream) {
    constexpr int kStages = 4;
    const size_t smem = kXbHeader + (size_t)kStages * kXbStageBytes;
    auto kernel = reduce_exact_bulk_kernel<kF16, true>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        static std::mutex mu;
        static std::map<int, size_t> configured;
        std::lock_guard<std::mutex> lk(mu);
        if (smem > configured[dev]) {
            if ((e = cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem)))
                return e;
            configured[dev] = smem;
        }
    }
    const int P = emulate ? pc.nranks : 1;
    const size_t C = n / (size_t)P * 2u / kXbStageBytes;
    size_t g = (size_t)cfg.sms / (size_t)P;
    if (g > C) g = C;
    if (g < 1) g = 1;
    const int dyn = (C >= (size_t)cfg.tc05_dyn_min_run * g) ? cfg.tc05_dynamic : 0;
    int stages = kStages;
    if (!emulate) {
        kernel<<<(unsigned)g, kXbThreads, smem, stream>>>(x, n, stages, dyn, out_acc, out_f32, out_f64, ws, pc);
        return cudaGetLastError();
    }
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kXbThreads, smem))) return e;
    const size_t cap = (size_t)occ * (size_t)cfg.sms / (size_t)P;
    if (g > cap) g = cap;
    if (g < 1) return cudaErrorCooperativeLaunchTooLarge;
    const uint8_t* xa = x;
    size_t na = n;
    long long* acc = out_acc;
    float* o32 = out_f32;
    double* o64 = out_f64;
    DevWorkspace wsa = ws;
    PeerCombine pca = pc;
    int dp = dyn;
    void* args[] = {(void*)&xa, (void*)&na, (void*)&stages, (void*)&dp, (void*)&acc, (void*)&o32,
                    (void*)&o64, (void*)&wsa, (void*)&pca};
    return cudaLaunchCooperativeKernel((const void*)kernel, dim3((unsigned)g, (unsigned)P), dim3(kXbThreads),
                                       args, smem, stream);
}

cudaError_t launch_reduce_exact_peer(const uint16_t* x, size_t n, long long* out_acc,
                                     float* out_f32, double* out_f64, const DevWorkspace& ws,
                                     const LaunchCfg& cfg, const PeerCombine& pc, bool emulate,
                                     cudaStream_t stream) {
    const int P0 = emulate ? pc.nranks : 1;
    const size_t shard_bytes = n / (size_t)(P0 > 0 ? P0 : 1) * 2u;
    // real ranks: the TMA-fed kernel from 128 MiB per rank (1 rank at 2^30: 300.9 vs 319.7 us);
    // emulated ranks share one GPU's SMs (one CTA per SM, SMs / P per rank), where the LDG
    // kernel's three CTAs per SM do better (8 x 2^30: 2553 vs 2800 us,
    // profiles/r02/exact_peer_ab.txt) -- forced with TCR_CFG_EXACT_BULK = 2
    if (cfg.exact_bulk == 2 || (cfg.exact_bulk == 1 && !emulate && shard_bytes >= ((size_t)128 << 20)))
        return launch_exact_bulk_peer(reinterpret_cast<const uint8_t*>(x), n, out_acc, out_f32, out_f64, ws,
                                      cfg, pc, emulate, stream);
    auto kernel = reduce_exact_kernel<8, true, kF16>;  // the peer variant: binary16, unroll 8
    LaunchCfg c8 = cfg;
    c8.exact_unroll = 8;
    if (!emulate) {
        const int g = exact_grid(n, c8, ws.capacity);
        kernel<<<g, kExactWarps * 32, 0, stream>>>(reinterpret_cast<const uint8_t*>(x), n, out_acc,
                                                   out_f32, out_f64, ws, pc);
        return cudaGetLastError();
    }
    // emulated ranks wait on one another: one cooperative launch (co-residency)
    const int P = pc.nranks;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kExactWarps * 32, 0);
    if (e != cudaSuccess) return e;
    int g = exact_grid(n / (size_t)P, c8, ws.capacity / P);
    const int cap = occ * cfg.sms / P;
    if (g > cap) g = cap;
    if (g < 1) return cudaErrorCooperativeLaunchTooLarge;
    const uint8_t* xa = reinterpret_cast<const uint8_t*>(x);
    size_t na = n;
    long long* acc = out_acc;
    float* o32 = out_f32;
    double* o64 = out_f64;
    DevWorkspace wsa = ws;
    PeerCombine pca = pc;
    void* args[] = {(void*)&xa, (void*)&na, (void*)&acc, (void*)&o32, (void*)&o64, (void*)&wsa,
                    (void*)&pca};
    return cudaLaunchCooperativeKernel((const void*)kernel, dim3(g, P), dim3(kExactWarps * 32),
                                       args, 0, stream);
}

cudaError_t launch_exact_finalize(const long long* acc, float* out_f32, double* out_f64,
                                  cudaStream_t stream) {
    exact_finalize_kernel<<<1, 32, 0, stream>>>(acc, out_f32, out_f64);
    return cudaGetLastError();
}

}  // namespace tcr
