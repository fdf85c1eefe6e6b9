// tcr_device.cuh -- device building blocks of the MMA-encoded reduction
// (sm_100a).  Citations "P:L" are lines of the paper text (arXiv 1903.03640).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace tcr {

constexpr int kTileElems = 256;  // one 16x16 fp16 MMA A operand = m^2 with m = 16
constexpr uint32_t kOnesH2 = 0x3C003C00u;  // two binary16 1.0: the all-ones B
constexpr uint32_t kOnesBf2 = 0x3F803F80u;  // two bfloat16 1.0 (NEXT-4 bfloat16 inputs)

// ---------------------------------------------------------------------------
// Loads
// ---------------------------------------------------------------------------

// Streaming 16-byte load: read-only path, no L1 allocation (every input is
// read exactly once), 256-byte L2 prefetch.  `volatile` keeps the issue
// order of the source: all U loads of an iteration are issued before the
// first MMA consumes one (ptxas otherwise interleaves them and the in-order
// issue stalls on the first consumer, leaving ~3 loads in flight per warp).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ uint16_t ldg_u16(const uint16_t* p) {
    uint16_t r;
    asm("ld.global.nc.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}

// ---------------------------------------------------------------------------
// Level 1: D = A x 1 + C  (Eq. 9-10) with mma.sync m16n8k16.
//
// A (16x16, row-major fragment): lane l = 4g + t holds a0..a3 = 8 halves.
// Loading the contiguous halves x[8l .. 8l+8) of a 256-element tile into
// a0..a3 is a bijection of the tile onto A (checked at index level in
// tests/test_fragment_layout.py); the reduction is permutation invariant,
// so this is a valid placement of the group into A (reading G1).
// B (16x8) = all ones.  D (16x8 fp32): c0 = c1 = row sum of row g,
// c2 = c3 = row sum of row g+8 (every column equal, Eq. 10).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_rowsum(float (&c)[4], const uint4& a) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(kOnesH2), "r"(kOnesH2));
}

// bfloat16 inputs (NEXT-4): the same encoding with .bf16 operands.
__device__ __forceinline__ void mma_rowsum_bf16(float (&c)[4], const uint4& a) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(kOnesBf2), "r"(kOnesBf2));
}

// Element formats of the flat reduction (NEXT-4): every one keeps the tile at
// 512 bytes = one 16-byte vector per lane.  An fp8 tile (512 elements, 16 per
// lane) is the A of an m16n8k32, issued as two m16n8k16 (below); the C/D
// fragment is unchanged.
enum Fmt : int { kF16 = 0, kBF16 = 1, kE4M3 = 2, kE5M2 = 3 };
template <int F> struct FmtInfo { static constexpr int kBytes = F >= kE4M3 ? 1 : 2; };

// fp8 tile as two binary16 A operands: every fp8 value is a binary16 value
// (cvt.rn.f16x2.{e4m3,e5m2}x2 is exact), so the 32 products of a row of the
// m16n8k32 become two m16n8k16 row sums against binary16 ones, chained in
// fp32 -- the same arithmetic ptxas emits for mma.sync m16n8k32.e4m3 on
// sm_100a (F2FP unpacks + two HMMA.16816), but converting only A: the
// instruction form re-converted the constant ones operand at every MMA and
// spilled at 80 registers (build/obj/tcr_reduce.ptxas.txt, r02).  Lane l's
// 16 bytes map to halves 0..7 of the first and second operand: a bijection
// of the tile onto A (reading G1).
template <int F>
__device__ __forceinline__ void mma_rowsum_fp8_as_f16(float (&c)[4], const uint4& a) {
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    uint32_t h[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint16_t lo = (uint16_t)(w[k] & 0xFFFFu), hi = (uint16_t)(w[k] >> 16);
        if constexpr (F == kE4M3) {
            asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h[2 * k]) : "h"(lo));
            asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h[2 * k + 1]) : "h"(hi));
        } else {
            asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h[2 * k]) : "h"(lo));
            asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h[2 * k + 1]) : "h"(hi));
        }
    }
    mma_rowsum(c, make_uint4(h[0], h[1], h[2], h[3]));
    mma_rowsum(c, make_uint4(h[4], h[5], h[6], h[7]));
}

template <int F>
__device__ __forceinline__ void mma_rowsum_f(float (&c)[4], const uint4& a) {
    if constexpr (F == kF16) mma_rowsum(c, a);
    else if constexpr (F == kBF16) mma_rowsum_bf16(c, a);
    else mma_rowsum_fp8_as_f16<F>(c, a);
}

// Flush the carried fp32 accumulator into the lane's fp64 accumulator and
// reset it (bounded chain, reading G9).  Rows g and g+8 appear in lanes
// 4g..4g+3 (c0 and c2); lane t==0 keeps row g, t==1 keeps row g+8, t>=2
// keep nothing, so the sum over lanes of `acc` is the sum over all 16 rows.
__device__ __forceinline__ void flush_rows(float (&c)[4], double& acc, int lane) {
    const int t = lane & 3;
    const float v = (t & 1) ? c[2] : c[0];
    acc += (t < 2) ? (double)v : 0.0;
    c[0] = c[1] = c[2] = c[3] = 0.0f;
}

// ---------------------------------------------------------------------------
// Level 2: D' = 1 x D (Eq. 11-12) on fp64 partials with three
// m8n8k4 DMMAs, A = all ones, "D in the position of B, ones in A".
// Input: one fp64 value v_l per lane.  Output (every lane): sum_l v_l.
//   DMMA 1: B[t][g] = v_{4g+t}     -> D[i][j] = S_j = sum_t v_{4j+t};
//           lane 4g+t holds d0 = S_{2t}, d1 = S_{2t+1}.
//   DMMA 2: B[t][g] = d0 of lane 4g+t = S_{2t} -> every entry sum of even S.
//   DMMA 3: B = d1 (S_{2t+1}), C = previous   -> every entry sum of all S.
// All 64 entries of the last D are the total: "the reduction of the m^2
// numbers, replicated in all of its elements".  Must be called by
// all 32 lanes (warp-synchronous).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_ones(double& d0, double& d1, double b, double c0, double c1) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
        : "=d"(d0), "=d"(d1)
        : "d"(1.0), "d"(b), "d"(c0), "d"(c1));
}

__device__ __forceinline__ double warp_collapse_mma(double v) {
    double s0, s1, e0, e1, f0, f1;
    dmma_ones(s0, s1, v, 0.0, 0.0);
    dmma_ones(e0, e1, s0, 0.0, 0.0);
    dmma_ones(f0, f1, s1, e0, e1);
    (void)f1;
    return f0;
}

// Classic comparison: butterfly tree with shfl_xor.
__device__ __forceinline__ double warp_collapse_shfl(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <bool kMma>
__device__ __forceinline__ double warp_collapse(double v) {
    if constexpr (kMma) return warp_collapse_mma(v);
    else return warp_collapse_shfl(v);
}

// ---------------------------------------------------------------------------
// Classic per-lane accumulation of one 16-byte vector (8 halves) in fp32.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float vec_sum_f32(const uint4& a) {
    const float2 p0 = __half22float2(*reinterpret_cast<const __half2*>(&a.x));
    const float2 p1 = __half22float2(*reinterpret_cast<const __half2*>(&a.y));
    const float2 p2 = __half22float2(*reinterpret_cast<const __half2*>(&a.z));
    const float2 p3 = __half22float2(*reinterpret_cast<const __half2*>(&a.w));
    return ((p0.x + p0.y) + (p1.x + p1.y)) + ((p2.x + p2.y) + (p3.x + p3.y));
}

// bfloat16 -> binary32 is exact: the bfloat16 is the top half of the binary32.
__device__ __forceinline__ float vec_sum_f32_bf16(const uint4& a) {
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    float p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = __uint_as_float(w[k] << 16) + __uint_as_float(w[k] & 0xFFFF0000u);
    return (p[0] + p[1]) + (p[2] + p[3]);
}

// fp8 -> binary16 pairs are exact (cvt.rn.f16x2.{e4m3,e5m2}x2), then binary32.
template <int F>
__device__ __forceinline__ float fp8x2_sum(uint16_t b) {
    uint32_t h2;
    if constexpr (F == kE4M3) asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(b));
    else asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(h2) : "h"(b));
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h2));
    return f.x + f.y;
}

template <int F>
__device__ __forceinline__ float vec_sum_f(const uint4& a) {
    if constexpr (F == kF16) return vec_sum_f32(a);
    else if constexpr (F == kBF16) return vec_sum_f32_bf16(a);
    else {
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
        float p[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            p[k] = fp8x2_sum<F>((uint16_t)(w[k] & 0xFFFFu)) + fp8x2_sum<F>((uint16_t)(w[k] >> 16));
        return (p[0] + p[1]) + (p[2] + p[3]);
    }
}

// A lane's 16 bytes of a ragged tile: bytes p[16*lane + k] for 16*lane + k <
// cnt_bytes, zero elsewhere (byte loads, never out of bounds).
__device__ __forceinline__ uint4 load_ragged_bytes(const uint8_t* p, int cnt_bytes, int lane) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int i = 16 * lane + k;
        if (i < cnt_bytes) w[k >> 2] |= (uint32_t)__ldg(p + i) << (8 * (k & 3));
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Zero the halves of a 16-byte vector whose element index (vector base
// `e0` + k) lies outside [lo, hi).
__device__ __forceinline__ uint4 mask_vec(uint4 v, int64_t e0, int64_t lo, int64_t hi) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i0 = e0 + 2 * k, i1 = i0 + 1;
        const uint32_t m0 = (i0 >= lo && i0 < hi) ? 0x0000FFFFu : 0u;
        const uint32_t m1 = (i1 >= lo && i1 < hi) ? 0xFFFF0000u : 0u;
        w[k] &= (m0 | m1);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// mask_vec for any element format: bytes of elements outside [lo, hi) zeroed
// (e0 = element index of the vector's first element).
template <int F>
__device__ __forceinline__ uint4 mask_vec_f(uint4 v, int64_t e0, int64_t lo, int64_t hi) {
    if constexpr (FmtInfo<F>::kBytes == 2) {
        return mask_vec(v, e0, lo, hi);
    } else {
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint32_t m = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int64_t i = e0 + 4 * k + b;
                if (i >= lo && i < hi) m |= 0xFFu << (8 * b);
            }
            w[k] &= m;
        }
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// A lane's 8 halves of a ragged (masked) tile: elements p[8*lane + k] for
// 8*lane + k < cnt, zero elsewhere; scalar loads, never out of bounds.
__device__ __forceinline__ uint4 load_ragged(const uint16_t* p, int cnt, int lane) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int i0 = 8 * lane + 2 * k, i1 = i0 + 1;
        const uint32_t lo = (i0 < cnt) ? (uint32_t)ldg_u16(p + i0) : 0u;
        const uint32_t hi = (i1 < cnt) ? (uint32_t)ldg_u16(p + i1) : 0u;
        w[k] = lo | (hi << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// ---------------------------------------------------------------------------
// Launch plumbing shared by the kernels (r02)
// ---------------------------------------------------------------------------

// Programmatic dependent launch (TCR_CFG_PDL): a kernel launched with the
// programmatic-serialisation attribute may be scheduled while the previous
// kernel on the stream drains.  griddepcontrol.wait blocks until that kernel
// has completed and its writes (x, the workspace's partials and counters) are
// visible; launch_dependents lets the next kernel be scheduled early in turn.
// Both are no-ops for a plain launch.  Call before touching global memory
// (CTA-local set-up -- barriers, TMEM allocation, SMEM tables -- may precede).
__device__ __forceinline__ void pdl_wait_and_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// Completion ticket: one acq_rel atomic at GPU scope.  Release orders the
// CTA's partial (stored by the same thread just before) ahead of the ticket;
// acquire makes every earlier CTA's partial visible to the last one (then
// __syncthreads() extends that to the whole CTA).  One atomic instead of
// __threadfence() + atomicAdd (~0.6 us less on the critical path,
// scripts/c2_trace.cu, profiles/r02/c2_trace_ab.txt).
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* t) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    return old;
}

// Host: launch `kernel` with the programmatic-serialisation attribute when
// pdl != 0 (cudaLaunchKernelEx; errors surface through cudaGetLastError).
template <typename... KArgs, typename... Args>
static inline void launch_maybe_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t stream, int pdl, Args... args) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&lc, kernel, static_cast<KArgs>(args)...);
}

}  // namespace tcr
