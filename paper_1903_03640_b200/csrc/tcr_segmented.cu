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

constexpr unsigned long long kBatchSeg = 8;  // segments per scheduler atomic (guided)

// Reduce elements [s, e) of the 16-byte-aligned array xb (element indices
// relative to xb).  Returns the lane's fp64 share; the sum over lanes is the
// segment total.
template <bool kMma, bool kBf16, int U>
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
                if (u & 1) mma_rowsum_t<kBf16>(cB, v[u]);
                else mma_rowsum_t<kBf16>(cA, v[u]);
            } else {
                if (u & 1) fB += vec_sum_t<kBf16>(v[u]);
                else fA += vec_sum_t<kBf16>(v[u]);
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

template <bool kMma, bool kBf16, bool kBatched, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4)
reduce_segmented_kernel(const uint16_t* __restrict__ x, const int64_t* __restrict__ offsets,
                        size_t S, size_t L, float* __restrict__ out, DevWorkspace ws) {
    const int lane = threadIdx.x & 31;
    const uintptr_t addr = (uintptr_t)x;
    const int64_t shift = (int64_t)((addr & 15u) >> 1);
    const uint4* xb = reinterpret_cast<const uint4*>(addr & ~(uintptr_t)15u);
    const unsigned total_warps = gridDim.x * WARPS;

    // Guided self-scheduling: a warp takes a batch of kBatchSeg consecutive
    // segments per atomic while plenty remain, single segments near the end
    // (one global atomic per segment saturates the L2 atomic unit at ~4 ns
    // per segment -- the whole C5 kernel time).
    const unsigned long long tail_zone = 2ull * total_warps * kBatchSeg;
    auto grab = [&](unsigned long long hint) -> unsigned long long {
        unsigned long long got = 0;
        const unsigned long long b = (S > hint + tail_zone) ? kBatchSeg : 1ull;
        if (lane == 0) got = atomicAdd(ws.seg_next, b) | (b << 56);
        return got;  // start index in bits 0..55, batch size in 56..63 (lane 0)
    };
    auto bounds = [&](unsigned long long jj, int64_t& ss, int64_t& ee) {
        if constexpr (kBatched) {
            ss = (int64_t)(jj * L);
            ee = ss + (int64_t)L;
        } else {
            ss = __ldg(offsets + jj);
            ee = __ldg(offsets + jj + 1);
        }
    };
    const unsigned long long kIdx = (1ull << 56) - 1;
    unsigned long long g = __shfl_sync(0xffffffffu, grab(0), 0);
    unsigned long long j = g & kIdx, batch_end = j + (g >> 56);
    int64_t s = 0, e = 0;
    if (j < S) bounds(j, s, e);
    while (j < S) {
        const bool last = (j + 1 == batch_end);
        unsigned long long gn = 0;
        if (last) gn = grab(j);  // next batch start, in flight during this segment
        const double acc = seg_reduce<kMma, kBf16, U>(xb, s + shift, e + shift, lane);
        unsigned long long jn;
        if (last) {
            gn = __shfl_sync(0xffffffffu, gn, 0);
            jn = gn & kIdx;
            batch_end = jn + (gn >> 56);
        } else {
            jn = j + 1;
        }
        int64_t sn = 0, en = 0;  // next bounds: their latency overlaps the collapse
        if (jn < S) bounds(jn, sn, en);
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

template <bool kMma, bool kBf16>
static void launch_seg_t(bool batched, const dim3& grid, const dim3& block, const uint16_t* x,
                         const int64_t* offsets, size_t S, size_t L, float* out,
                         const DevWorkspace& ws, cudaStream_t stream) {
    if (batched)
        reduce_segmented_kernel<kMma, kBf16, true, kSegUnroll, kSegWarps>
            <<<grid, block, 0, stream>>>(x, offsets, S, L, out, ws);
    else
        reduce_segmented_kernel<kMma, kBf16, false, kSegUnroll, kSegWarps>
            <<<grid, block, 0, stream>>>(x, offsets, S, L, out, ws);
}

cudaError_t launch_reduce_segmented(bool mma, bool bf16, bool batched, const uint16_t* x,
                                    const int64_t* offsets, size_t num_segments,
                                    size_t segment_len, float* out, const DevWorkspace& ws,
                                    const LaunchCfg& cfg, cudaStream_t stream) {
    size_t g = (num_segments + kSegWarps - 1) / kSegWarps;
    const size_t gmax = (size_t)cfg.sms * kSegCtasPerSm;
    if (g > gmax) g = gmax;
    if (g < 1) g = 1;
    const dim3 grid((unsigned)g), block(kSegWarps * 32);
    if (mma) {
        if (bf16) launch_seg_t<true, true>(batched, grid, block, x, offsets, num_segments, segment_len, out, ws, stream);
        else launch_seg_t<true, false>(batched, grid, block, x, offsets, num_segments, segment_len, out, ws, stream);
    } else {
        if (bf16) launch_seg_t<false, true>(batched, grid, block, x, offsets, num_segments, segment_len, out, ws, stream);
        else launch_seg_t<false, false>(batched, grid, block, x, offsets, num_segments, segment_len, out, ws, stream);
    }
    return cudaGetLastError();
}

}  // namespace tcr
