// tcr_reduce.cu -- the streaming MMA-encoded reduction (mma.sync m16n8k16,
// 128-bit loads) and its classic warp-shuffle twin, with last-CTA grid
// completion.  One launch computes the whole hierarchy R_tc of the paper
// (Eq. 13-14):
//
//   level 1  tile:  D = A x 1 + C, 256 inputs -> 16 row sums   (Eq. 9-10)
//                   C carried over a bounded chain of K tiles,
//                   then flushed into a per-lane fp64 accumulator
//   level 2  warp:  D' = 1 x D via three fp64 DMMAs            (Eq. 11-12)
//   level 3  CTA:   the same 1 x D collapse over the warp totals
//   level 4  grid:  last CTA (completion ticket) collapses the CTA partials
//                   in index order -- replaces the paper's relaunch per level
//                   ("synchronization among blocks is not possible ... unless
//                   the kernel is terminated").
#include "tcr_complete.cuh"
#include "tcr_device.cuh"
#include "tcr_internal.h"

namespace tcr {

template <bool kMma, int F>
__device__ __forceinline__ void consume(const uint4& v, float (&c)[4], float& f) {
    if constexpr (kMma) mma_rowsum_f<F>(c, v);
    else f += vec_sum_f<F>(v);
}

template <bool kMma>
__device__ __forceinline__ void flush(float (&c)[4], float& f, double& acc, int lane) {
    if constexpr (kMma) flush_rows(c, acc, lane);
    else { acc += (double)f; f = 0.0f; }
}

// The U vectors of one batch, alternately into the two accumulators.  With
// mid_flush (U = 16 at the default chain K = 4) both are flushed after the
// first half of the batch, so no accumulator carries more than K tiles.
template <bool kMma, int F, int U>
__device__ __forceinline__ void consume_batch(const uint4 (&v)[U], float (&cA)[4], float (&cB)[4],
                                              float& fA, float& fB, double& acc, int lane,
                                              bool mid_flush) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (u & 1) consume<kMma, F>(v[u], cB, fB);
        else consume<kMma, F>(v[u], cA, fA);
        if (U == 16 && u == U / 2 - 1 && mid_flush) {
            flush<kMma>(cA, fA, acc, lane);
            flush<kMma>(cB, fB, acc, lane);
        }
    }
}

// Grid-stride over 512-byte tiles: warp w handles tiles w, w+W, w+2W, ...,
// U tiles (one 16-byte vector per lane each) in flight per iteration.
// __launch_bounds__ minimum CTAs/SM: without it ptxas budgets registers for
// full occupancy (32 regs at 256 threads) and sinks the U loads below their
// consumers, which leaves ~2 loads in flight per warp.  F = element format
// (binary16, bfloat16, fp8 E4M3 / E5M2); all index math is in bytes.
// kPeer: the NEXT-2 variant (fused cross-GPU combine, tcr_peer.cuh; grid.y
// slices = emulated ranks).  A separate instantiation, so that the plain
// kernel's code is untouched by it (measured: folding the peer path into
// the plain kernel as a runtime branch cost 3 % at 2^30).
// Resident CTAs per SM the register budget is sized for (__launch_bounds__):
// 4 at U <= 8 (64 registers), 2 at U = 16 -- every format at zero spills
// (build/obj/tcr_reduce.ptxas.txt).
template <int F, int U>
constexpr int stream_resident() { return U <= 8 ? 4 : 2; }

template <bool kMma, int F, int U, int WARPS, bool kPeer>
__global__ void __launch_bounds__(WARPS * 32, stream_resident<F, U>())
reduce_stream_kernel(const uint8_t* __restrict__ x, size_t n, int flush_every, int mid_flush,
                     float* out_f32, double* out_f64, DevWorkspace ws, PeerCombine pc) {
    constexpr int ES = FmtInfo<F>::kBytes;
    constexpr int kTileBytes = 512;
    TCR_COMPLETE_EDGE(0);
    // Programmatic dependent launch (TCR_CFG_PDL): this grid may have been
    // scheduled while the previous kernel on the stream drained; wait for it
    // to complete (and its writes -- x, the workspace -- to be visible)
    // before touching memory, then let the next call's grid be scheduled.
    // Both are no-ops for a plain launch.
    pdl_wait_and_release();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int me = pc.rank;
    if (kPeer && gridDim.y > 1) {  // emulated peer group: slice y is rank y, reducing its shard
        const size_t P = gridDim.y, r = blockIdx.y;
        const size_t lo = r * n / P, hi = (r + 1) * n / P;
        x += lo * ES;
        n = hi - lo;
        ws.partials += r * gridDim.x;
        ws.ticket += r;
        if (out_f32) out_f32 += r;
        if (out_f64) out_f64 += r;
        me = (int)r;
    }
    const size_t nbytes = n * ES;
    // head: bytes before the first 16-byte boundary (x is element aligned)
    size_t head = (16u - ((uintptr_t)x & 15u)) & 15u;
    if (head > nbytes) head = nbytes;
    const uint8_t* xa = x + head;
    const size_t nb = nbytes - head;
    const size_t T = nb / kTileBytes;
    const int tail = (int)(nb - T * kTileBytes);
    const size_t W = (size_t)gridDim.x * WARPS;
    const size_t w = (size_t)blockIdx.x * WARPS + warp;
    const uint4* base = reinterpret_cast<const uint4*>(xa) + lane;

    double acc = 0.0;
    float cA[4] = {0.f, 0.f, 0.f, 0.f}, cB[4] = {0.f, 0.f, 0.f, 0.f};
    float fA = 0.f, fB = 0.f;
    int it = 0;
    size_t t = w;
    for (; t + (size_t)(U - 1) * W < T; t += (size_t)U * W) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream(base + (t + (size_t)u * W) * 32);
        __syncwarp();  // scheduling fence: all U loads issue before the first consumer
        consume_batch<kMma, F, U>(v, cA, cB, fA, fB, acc, lane, mid_flush != 0);
        if (++it == flush_every) {
            it = 0;
            flush<kMma>(cA, fA, acc, lane);
            flush<kMma>(cB, fB, acc, lane);
        }
    }
    if (t < T) {  // fewer than U tiles left for this warp: one predicated batch
        // (all loads in flight together -- one latency, not one per tile;
        // a zero vector adds exactly nothing)
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            v[u] = (t + (size_t)u * W < T) ? ldg_stream(base + (t + (size_t)u * W) * 32)
                                           : make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        consume_batch<kMma, F, U>(v, cA, cB, fA, fB, acc, lane, mid_flush != 0);
    }
    flush<kMma>(cA, fA, acc, lane);
    flush<kMma>(cB, fB, acc, lane);
    if (w == W - 1) {  // ragged head and tail: zero-padded tiles (reading G5)
        if (head) {
            consume<kMma, F>(load_ragged_bytes(x, (int)head, lane), cA, fA);
            flush<kMma>(cA, fA, acc, lane);
        }
        if (tail) {
            consume<kMma, F>(load_ragged_bytes(xa + T * kTileBytes, tail, lane), cA, fA);
            flush<kMma>(cA, fA, acc, lane);
        }
    }
    TCR_COMPLETE_EDGE(2);
    complete_block_and_grid<kMma, WARPS>(acc, out_f32, out_f64, ws, kPeer ? &pc : nullptr, me);
    TCR_COMPLETE_EDGE(3);
}

constexpr int kStreamWarps = 8;  // 256 threads per CTA

int stream_grid(size_t n, const LaunchCfg& cfg, int resident_in) {
    const size_t tiles = n / kTileElems;  // (n in 2-byte element equivalents)
    const size_t per_cta = (size_t)kStreamWarps * cfg.unroll;  // tiles one CTA covers per iteration
    size_t g = (tiles + per_cta - 1) / per_cta;
    // Large inputs (HBM-bound): oversubscribe with blocks_per_sm CTAs per SM
    // (measured best at 2^30).  Below 2^28 elements the launch is latency
    // bound and a second wave costs more than it hides: cap the grid at one
    // resident wave (the __launch_bounds__ minimum CTAs per SM).
    const int resident = resident_in > 0 ? resident_in : (cfg.unroll <= 8 ? 4 : 2);
    const int per_sm = (n < ((size_t)1 << 28) && cfg.blocks_per_sm > resident) ? resident
                                                                               : cfg.blocks_per_sm;
    const size_t gmax = (size_t)cfg.sms * per_sm;
    if (g > gmax) g = gmax;
    // Up to two load rounds of work: one CTA, no grid completion -- the
    // ticket + last-CTA pass costs more than a second round of loads
    // (2^16 elements: 2.87 vs 3.51 us, scripts/runs/ab_small.py).
    if (tiles <= 2 * per_cta) g = 1;
    if (g < 1) g = 1;
    return (int)g;
}

template <bool kMma, int F, int U, bool kPeer>
static cudaError_t launch_stream_u(const uint8_t* x, size_t n, int fe, float* out_f32,
                                   double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                   const PeerCombine& pc, bool emulate, cudaStream_t stream) {
    auto kernel = reduce_stream_kernel<kMma, F, U, kStreamWarps, kPeer>;
    const int mid = (U == 16 && 2 * cfg.chain < U) ? 1 : 0;
    if (!emulate) {
        const int g = stream_grid(n * FmtInfo<F>::kBytes / 2, cfg, stream_resident<F, U>());
        // (the peer variant waits on other ranks: plain launch)
        launch_maybe_pdl(kernel, dim3(g), dim3(kStreamWarps * 32), 0, stream, (cfg.pdl && !kPeer) ? 1 : 0,
                         x, n, fe, mid, out_f32, out_f64, ws, pc);
        return cudaGetLastError();
    }
    // Emulated peer group: the ranks' last CTAs wait on one another, so all
    // P grid slices must be co-resident -- a cooperative launch guarantees it
    // (B200_PROFILING.md: emulate ranks as one kernel, never as separate launches).
    const int P = pc.nranks;
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kStreamWarps * 32, 0);
    if (e != cudaSuccess) return e;
    int g = stream_grid(n / (size_t)P * FmtInfo<F>::kBytes / 2, cfg);
    const int cap = occ * cfg.sms / P;
    if (g > cap) g = cap;
    if (g < 1) return cudaErrorCooperativeLaunchTooLarge;
    const uint8_t* xa = x;
    size_t na = n;
    int fea = fe, mida = mid;
    float* o32 = out_f32;
    double* o64 = out_f64;
    DevWorkspace wsa = ws;
    PeerCombine pca = pc;
    void* args[] = {(void*)&xa, (void*)&na, (void*)&fea, (void*)&mida, (void*)&o32, (void*)&o64,
                    (void*)&wsa, (void*)&pca};
    return cudaLaunchCooperativeKernel((const void*)kernel, dim3(g, P), dim3(kStreamWarps * 32),
                                       args, 0, stream);
}

// Inputs below this many 2-byte element equivalents are latency bound: the
// auto unroll (TCR_CFG_UNROLL = 0) puts 16 loads per lane in flight there
// (one or two load rounds per warp instead of four; -0.4 to -0.7 us at
// 2^22..2^25, profiles/r01/c2_sweep2.txt) and 4 above (the measured best
// at 2^30).
constexpr size_t kSmallN = (size_t)1 << 26;

template <bool kMma, int F>
static cudaError_t launch_stream_t(const uint16_t* x16, size_t n, float* out_f32, double* out_f64,
                                   const DevWorkspace& ws, const LaunchCfg& cfg_in,
                                   const PeerCombine& pc, bool emulate, cudaStream_t stream) {
    const uint8_t* x = reinterpret_cast<const uint8_t*>(x16);
    LaunchCfg cfg = cfg_in;
    if (pc.nranks > 0) {
        // the peer variant is instantiated at unroll 4 only (build size)
        cfg.unroll = 4;
        const int fe = 2 * cfg.chain / 4 < 1 ? 1 : 2 * cfg.chain / 4;
        return launch_stream_u<kMma, F, 4, true>(x, n, fe, out_f32, out_f64, ws, cfg, pc, emulate,
                                                 stream);
    }
    if (cfg.unroll == 0) cfg.unroll = (n * FmtInfo<F>::kBytes / 2 < kSmallN) ? 16 : 4;
    // two interleaved accumulators take unroll/2 tiles each per iteration
    const int fe = 2 * cfg.chain / cfg.unroll < 1 ? 1 : 2 * cfg.chain / cfg.unroll;
    switch (cfg.unroll) {
        case 4:
            return launch_stream_u<kMma, F, 4, false>(x, n, fe, out_f32, out_f64, ws, cfg, pc,
                                                      false, stream);
        case 16:
            return launch_stream_u<kMma, F, 16, false>(x, n, fe, out_f32, out_f64, ws, cfg, pc,
                                                       false, stream);
        default:
            return launch_stream_u<kMma, F, 8, false>(x, n, fe, out_f32, out_f64, ws, cfg, pc,
                                                      false, stream);
    }
}

template <int F>
static cudaError_t launch_stream_f(bool mma, const uint16_t* x, size_t n, float* out_f32,
                                   double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                   const PeerCombine& pc, bool emulate, cudaStream_t stream) {
    return mma ? launch_stream_t<true, F>(x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream)
               : launch_stream_t<false, F>(x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream);
}

cudaError_t launch_reduce_stream_peer(bool mma, int fmt, const uint16_t* x, size_t n,
                                      float* out_f32, double* out_f64, const DevWorkspace& ws,
                                      const LaunchCfg& cfg, const PeerCombine& pc, bool emulate,
                                      cudaStream_t stream) {
    switch (fmt) {
        case kBF16:
            return launch_stream_f<kBF16>(mma, x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream);
        case kE4M3:
            return launch_stream_f<kE4M3>(mma, x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream);
        case kE5M2:
            return launch_stream_f<kE5M2>(mma, x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream);
        default:
            return launch_stream_f<kF16>(mma, x, n, out_f32, out_f64, ws, cfg, pc, emulate, stream);
    }
}

cudaError_t launch_reduce_stream(bool mma, int fmt, const uint16_t* x, size_t n, float* out_f32,
                                 double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                 cudaStream_t stream) {
    PeerCombine none{};
    return launch_reduce_stream_peer(mma, fmt, x, n, out_f32, out_f64, ws, cfg, none, false, stream);
}

// ---------------------------------------------------------------------------
// Small kernels: combine of chunk partials (host entry), f64 -> f32 rounding
// (sharded finaliser), and the MMA rounding probe.
// ---------------------------------------------------------------------------

// One warp: lane l sums partials l, l+32, ... in order, then 1 x D collapse.
__global__ void sum_partials_kernel(const double* __restrict__ p, size_t count, float* out_f32,
                                    double* out_f64) {
    const int lane = threadIdx.x & 31;
    double v = 0.0;
    for (size_t i = lane; i < count; i += 32) v += p[i];
    const double tot = warp_collapse_mma(v);
    if (lane == 0) {
        if (out_f32) *out_f32 = (float)tot;
        if (out_f64) *out_f64 = tot;
    }
}

cudaError_t launch_sum_partials(const double* partials, size_t count, float* out_f32,
                                double* out_f64, cudaStream_t stream) {
    sum_partials_kernel<<<1, 32, 0, stream>>>(partials, count, out_f32, out_f64);
    return cudaGetLastError();
}

__global__ void round_f64_kernel(const double* in, float* out) {
    if (threadIdx.x == 0) *out = (float)*in;
}

cudaError_t launch_round_f64(const double* in, float* out, cudaStream_t stream) {
    round_f64_kernel<<<1, 32, 0, stream>>>(in, out);
    return cudaGetLastError();
}

// One m16n8k16 with A = a (row-major 16x16), B = ones, C[r][*] = c[r];
// writes column 0 of D (d[r] = D[r][0]).  Lane 4g+t: a0 = A[g][2t..2t+1],
// a1 = A[g+8][2t..], a2 = A[g][2t+8..], a3 = A[g+8][2t+8..] (PTX ISA
// fragment layout of m16n8k16 .f16 A); c0 = C[g][2t], c2 = C[g+8][2t].
__global__ void probe_mma_sync_kernel(const uint16_t* a, const float* c, float* d) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    auto pack = [&](int r, int k) {
        return (uint32_t)a[r * 16 + k] | ((uint32_t)a[r * 16 + k + 1] << 16);
    };
    const uint4 av = make_uint4(pack(g, 2 * t), pack(g + 8, 2 * t), pack(g, 2 * t + 8),
                                pack(g + 8, 2 * t + 8));
    float acc[4] = {c[g], c[g], c[g + 8], c[g + 8]};
    mma_rowsum(acc, av);
    if (t == 0) {
        d[g] = acc[0];
        d[g + 8] = acc[2];
    }
}

cudaError_t launch_probe_mma_sync(const uint16_t* a, const float* c, float* d,
                                  cudaStream_t stream) {
    probe_mma_sync_kernel<<<1, 32, 0, stream>>>(a, c, d);
    return cudaGetLastError();
}

// Level-2 collapse probe: lane l holds in[l]; out[l] = the lane's result of
// warp_collapse (three DMMAs with ones in A, or the shfl_xor tree).
__global__ void probe_collapse_kernel(const double* in, double* out, int mma) {
    const int lane = threadIdx.x & 31;
    out[lane] = mma ? warp_collapse_mma(in[lane]) : warp_collapse_shfl(in[lane]);
}

cudaError_t launch_probe_collapse(const double* in, double* out, bool mma, cudaStream_t stream) {
    probe_collapse_kernel<<<1, 32, 0, stream>>>(in, out, mma ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace tcr
