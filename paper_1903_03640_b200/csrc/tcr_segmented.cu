// tcr_segmented.cu -- per-segment MMA-encoded reduction (CSR offsets or
// fixed-length batches).  One warp reduces one whole segment: level 1
// (D = A x 1 + C over 256-element tiles, Eq. 9-10) with the segment's
// unaligned head and tail zero-masked inside the tile (the paper's zero
// padding of the trailing group, reading G5), then level 2 (D' = 1 x D,
// Eq. 11-12) writes out[j].  Segments are owned whole, so there is no grid
// completion; warps take segments from a self-resetting counter (dynamic
// load balance for the log-uniform length mix).
#include "tcr_device.cuh"
#include "tcr_internal.h"

namespace tcr {

// Reduce elements [s, e) of the 16-byte-aligned array xb (element indices
// relative to xb).  Returns the lane's fp64 share; the sum over lanes is the
// segment total.
template <bool kMma, int U>
__device__ __forceinline__ double seg_reduce(const uint4* __restrict__ xb, int64_t s, int64_t e,
                                             int lane) {
    double acc = 0.0;
    if (e <= s) return acc;
    float cA[4] = {0.f, 0.f, 0.f, 0.f}, cB[4] = {0.f, 0.f, 0.f, 0.f};
    float fA = 0.f, fB = 0.f;
    const int64_t v0 = s >> 3, v1 = (e + 7) >> 3;  // vectors touching [s, e)
    const int64_t f0 = (s + 7) >> 3, f1 = e >> 3;  // vectors entirely inside
    // Every group of U tiles (32*U vectors) is one memory round trip: interior
    // groups load unmasked; the first and last groups load only the vectors
    // that touch the segment (predicated) and zero the halves outside it.
    for (int64_t vb = v0; vb < v1; vb += 32 * U) {
        uint4 v[U];
        if (vb >= f0 && vb + 32 * U <= f1) {
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ldg_stream(xb + vb + u * 32 + lane);
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t vi = vb + u * 32 + lane;
                v[u] = make_uint4(0u, 0u, 0u, 0u);
                if (vi < v1) v[u] = mask_vec(ldg_stream(xb + vi), vi * 8, s, e);
            }
        }
        __syncwarp();  // scheduling fence: all U loads issue before the first consumer
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if constexpr (kMma) {
                if (u & 1) mma_rowsum(cB, v[u]);
                else mma_rowsum(cA, v[u]);
            } else {
                if (u & 1) fB += vec_sum_f32(v[u]);
                else fA += vec_sum_f32(v[u]);
            }
        }
        if constexpr (kMma) {
            flush_rows(cA, acc, lane);
            flush_rows(cB, acc, lane);
        } else {
            acc += (double)fA + (double)fB;
            fA = fB = 0.f;
        }
    }
    return acc;
}

template <bool kMma, bool kBatched, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4)
reduce_segmented_kernel(const uint16_t* __restrict__ x, const int64_t* __restrict__ offsets,
                        size_t S, size_t L, float* __restrict__ out, DevWorkspace ws) {
    const int lane = threadIdx.x & 31;
    const uintptr_t addr = (uintptr_t)x;
    const int64_t shift = (int64_t)((addr & 15u) >> 1);
    const uint4* xb = reinterpret_cast<const uint4*>(addr & ~(uintptr_t)15u);
    const unsigned total_warps = gridDim.x * WARPS;

    unsigned long long j = 0;
    if (lane == 0) j = atomicAdd(ws.seg_next, 1ull);
    j = __shfl_sync(0xffffffffu, j, 0);
    int64_t s = 0, e = 0;
    if (j < S) {
        if constexpr (kBatched) {
            s = (int64_t)(j * L);
            e = s + (int64_t)L;
        } else {
            s = __ldg(offsets + j);
            e = __ldg(offsets + j + 1);
        }
    }
    while (j < S) {
        unsigned long long jn = 0;
        if (lane == 0) jn = atomicAdd(ws.seg_next, 1ull);  // next segment index, in flight
        const double acc = seg_reduce<kMma, U>(xb, s + shift, e + shift, lane);
        // the next index has arrived by now; start loading its offsets before
        // the collapse so that their latency overlaps it
        jn = __shfl_sync(0xffffffffu, jn, 0);
        int64_t sn = 0, en = 0;
        if (jn < S) {
            if constexpr (kBatched) {
                sn = (int64_t)(jn * L);
                en = sn + (int64_t)L;
            } else {
                sn = __ldg(offsets + jn);
                en = __ldg(offsets + jn + 1);
            }
        }
        const double tot = warp_collapse<kMma>(acc);
        if (lane == 0) out[j] = (float)tot;
        j = jn;
        s = sn;
        e = en;
    }
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(ws.seg_exit, 1u) == total_warps - 1) {  // last warp out resets the scheduler
            *ws.seg_next = 0ull;
            *ws.seg_exit = 0u;
            __threadfence();
        }
    }
}

constexpr int kSegWarps = 8;
constexpr int kSegUnroll = 8;
constexpr int kSegCtasPerSm = 4;  // resident CTAs per SM at <= 64 registers (launch bounds)

cudaError_t launch_reduce_segmented(bool mma, bool batched, const uint16_t* x,
                                    const int64_t* offsets, size_t num_segments,
                                    size_t segment_len, float* out, const DevWorkspace& ws,
                                    const LaunchCfg& cfg, cudaStream_t stream) {
    size_t g = (num_segments + kSegWarps - 1) / kSegWarps;
    const size_t gmax = (size_t)cfg.sms * kSegCtasPerSm;
    if (g > gmax) g = gmax;
    if (g < 1) g = 1;
    const dim3 grid((unsigned)g), block(kSegWarps * 32);
    if (mma) {
        if (batched)
            reduce_segmented_kernel<true, true, kSegUnroll, kSegWarps>
                <<<grid, block, 0, stream>>>(x, offsets, num_segments, segment_len, out, ws);
        else
            reduce_segmented_kernel<true, false, kSegUnroll, kSegWarps>
                <<<grid, block, 0, stream>>>(x, offsets, num_segments, segment_len, out, ws);
    } else {
        if (batched)
            reduce_segmented_kernel<false, true, kSegUnroll, kSegWarps>
                <<<grid, block, 0, stream>>>(x, offsets, num_segments, segment_len, out, ws);
        else
            reduce_segmented_kernel<false, false, kSegUnroll, kSegWarps>
                <<<grid, block, 0, stream>>>(x, offsets, num_segments, segment_len, out, ws);
    }
    return cudaGetLastError();
}

}  // namespace tcr
