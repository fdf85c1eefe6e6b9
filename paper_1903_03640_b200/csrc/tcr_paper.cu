// tcr_paper.cu -- the paper's algorithm taken literally (§IV.A),
// as a STUDY mode for NEXT-1 (precision) and for measuring the design change
// "one launch, not one per level".  Not the product path.
//
//   level kernel: one warp per group of m^2 = 256 inputs (zero-padded, G5):
//     D  = A x 1 + 0            mma.sync m16n8k16 .f16.f16.f16.f16 (Eq. 9-10,
//                               "A x B + C are done in FP16")
//     D' = 1 x D + 0            the row sums of D moved into B (shuffles),
//                               ones in A, again fp16 (Eq. 11-12)
//     X'[g] = D'_{1,1}          written to memory as binary16
//   host: relaunch on the n/256 partials until one value is left (Eq. 13-14,
//   "the kernel is terminated" between levels).
// Everything is binary16: the accumulate, the partials, the recursion.
#include "tcr_device.cuh"
#include "tcr_internal.h"

namespace tcr {

namespace {

__device__ __forceinline__ void mma_f16acc(uint32_t& d0, uint32_t& d1, const uint4& a, uint32_t b0,
                                           uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 "
                 "{%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%9};"
                 : "=r"(d0), "=r"(d1)
                 : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1), "r"(0u), "r"(0u));
}

constexpr int kLevelWarps = 8;

__global__ void __launch_bounds__(kLevelWarps * 32)
paper_level_kernel(const uint16_t* __restrict__ in, size_t len, uint16_t* __restrict__ out,
                   float* out_f32) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const size_t groups = (len + kTileElems - 1) / kTileElems;
    const size_t W = (size_t)gridDim.x * kLevelWarps;
    const bool aligned16 = ((uintptr_t)in & 15u) == 0;
    for (size_t grp = (size_t)blockIdx.x * kLevelWarps + (threadIdx.x >> 5); grp < groups; grp += W) {
        const uint16_t* p = in + grp * kTileElems;
        const size_t left = len - grp * kTileElems;
        const int cnt = left < (size_t)kTileElems ? (int)left : kTileElems;
        const uint4 a = (aligned16 && cnt == kTileElems)
                            ? ldg_stream(reinterpret_cast<const uint4*>(p) + lane)
                            : load_ragged(p, cnt, lane);
        uint32_t d0, d1;  // row sums: d0 = (R_g, R_g), d1 = (R_{g+8}, R_{g+8}) (fp16)
        mma_f16acc(d0, d1, a, kOnesH2, kOnesH2);
        // B[k][j] = R_k for the second MMA: lane (g, t) needs R_{2t}, R_{2t+1},
        // R_{2t+8}, R_{2t+9}; R_r sits in lanes 4r.. (d0) and R_{r+8} in d1 there.
        const uint32_t v0 = __shfl_sync(0xffffffffu, d0, 8 * t);
        const uint32_t v1 = __shfl_sync(0xffffffffu, d0, 8 * t + 4);
        const uint32_t v2 = __shfl_sync(0xffffffffu, d1, 8 * t);
        const uint32_t v3 = __shfl_sync(0xffffffffu, d1, 8 * t + 4);
        const uint32_t b0 = (v0 & 0xFFFFu) | (v1 << 16);
        const uint32_t b1 = (v2 & 0xFFFFu) | (v3 << 16);
        const uint4 ones = make_uint4(kOnesH2, kOnesH2, kOnesH2, kOnesH2);
        uint32_t e0, e1;  // D' = 1 x D: the group total in every entry (Eq. 12)
        mma_f16acc(e0, e1, ones, b0, b1);
        (void)g;
        (void)e1;
        if (lane == 0) {
            out[grp] = (uint16_t)(e0 & 0xFFFFu);  // D'_{1,1}
            if (out_f32 && groups == 1) *out_f32 = __half2float(__ushort_as_half((uint16_t)e0));
        }
    }
}

// ---------------------------------------------------------------------------
// NEXT-1 comparison points (study mode): the classic reduction entirely in
// binary32 -- naive, or with Kahan compensation at the lane and grid levels
// (A13) -- with the same loads, tree shape and last-CTA completion as the
// product's shuffle path but no fp64 anywhere.
// ---------------------------------------------------------------------------
template <bool kKahan>
__device__ __forceinline__ void add_f32(float& s, float& c, float v) {
    if constexpr (kKahan) {
        const float y = v - c;
        const float t = s + y;
        c = (t - s) - y;
        s = t;
    } else {
        s += v;
    }
}

template <bool kKahan>
__global__ void __launch_bounds__(kLevelWarps * 32)
study_fp32_kernel(const uint16_t* __restrict__ x, size_t n, float* out, DevWorkspace ws) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    size_t head = ((16u - ((uintptr_t)x & 15u)) & 15u) >> 1;
    if (head > n) head = n;
    const uint16_t* xa = x + head;
    const size_t nb = n - head;
    const size_t T = nb / kTileElems;
    const int tail = (int)(nb - T * kTileElems);
    const size_t W = (size_t)gridDim.x * kLevelWarps;
    const size_t w = (size_t)blockIdx.x * kLevelWarps + warp;
    const uint4* base = reinterpret_cast<const uint4*>(xa) + lane;
    float s = 0.f, c = 0.f;
    size_t t = w;
    for (; t + 3 * W < T; t += 4 * W) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = ldg_stream(base + (t + (size_t)u * W) * 32);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 4; ++u) add_f32<kKahan>(s, c, vec_sum_f32(v[u]));
    }
    for (; t < T; t += W) add_f32<kKahan>(s, c, vec_sum_f32(ldg_stream(base + t * 32)));
    if (w == W - 1) {
        if (head) add_f32<kKahan>(s, c, vec_sum_f32(load_ragged(x, (int)head, lane)));
        if (tail) add_f32<kKahan>(s, c, vec_sum_f32(load_ragged(xa + T * kTileElems, tail, lane)));
    }
    float v = s;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // binary32 tree
    __shared__ float s_warp[kLevelWarps];
    __shared__ unsigned s_last;
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    if (warp != 0) return;
    float b = lane < kLevelWarps ? s_warp[lane] : 0.f;
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    float* parts = reinterpret_cast<float*>(ws.partials);
    if (lane == 0) {
        parts[blockIdx.x] = b;
        __threadfence();
        s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
    __syncwarp();
    if (!s_last) return;
    if (lane == 0) {
        __threadfence();
        float gs = 0.f, gc = 0.f;
        for (unsigned i = 0; i < gridDim.x; ++i) add_f32<kKahan>(gs, gc, __ldcg(parts + i));
        *out = gs;
        *ws.ticket = 0u;
    }
}

}  // namespace

cudaError_t launch_study_fp32(const uint16_t* x, size_t n, bool kahan, float* out,
                              const DevWorkspace& ws, int sms, cudaStream_t stream) {
    const size_t tiles = n / kTileElems;
    size_t g = (tiles + 4 * kLevelWarps - 1) / (4 * kLevelWarps);
    const size_t gmax = (size_t)sms * 4;
    if (g > gmax) g = gmax;
    if (g > (size_t)ws.capacity) g = ws.capacity;
    if (g < 1) g = 1;
    if (kahan)
        study_fp32_kernel<true><<<(unsigned)g, kLevelWarps * 32, 0, stream>>>(x, n, out, ws);
    else
        study_fp32_kernel<false><<<(unsigned)g, kLevelWarps * 32, 0, stream>>>(x, n, out, ws);
    return cudaGetLastError();
}

size_t paper_scratch_elems(size_t n) {
    size_t total = 0;
    for (size_t len = n; len > 1;) {
        len = (len + kTileElems - 1) / kTileElems;
        total += len;
    }
    return total + 1;
}

cudaError_t launch_reduce_paper_f16(const uint16_t* x, size_t n, uint16_t* scratch, float* out_f32,
                                    int sms, cudaStream_t stream, int* launches) {
    *launches = 0;
    if (n == 0) {
        // R(empty) = +0.0 (G5): one level over a zero-length input writes nothing; do it here
        cudaError_t e = cudaMemsetAsync(out_f32, 0, sizeof(float), stream);
        return e;
    }
    const uint16_t* in = x;
    size_t len = n;
    uint16_t* dst = scratch;
    do {
        const size_t groups = (len + kTileElems - 1) / kTileElems;
        size_t g = (groups + kLevelWarps - 1) / kLevelWarps;
        const size_t gmax = (size_t)sms * 8;
        if (g > gmax) g = gmax;
        paper_level_kernel<<<(unsigned)g, kLevelWarps * 32, 0, stream>>>(in, len, dst,
                                                                         groups == 1 ? out_f32
                                                                                     : nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
        in = dst;
        dst += groups;
        len = groups;
    } while (len > 1);
    return cudaSuccess;
}

}  // namespace tcr
