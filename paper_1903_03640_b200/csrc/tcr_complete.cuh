// tcr_complete.cuh -- levels 2-4 of the in-kernel R_tc hierarchy, shared by
// the MMA kernels: warp collapse (D' = 1 x D, Eq. 11-12), CTA combine, and
// the grid level through a last-CTA completion ticket -- the replacement for
// the paper's kernel relaunch per level.
#pragma once

#include "tcr_device.cuh"
#include "tcr_internal.h"
#include "tcr_peer.cuh"

#ifndef TCR_COMPLETE_EDGE
#define TCR_COMPLETE_EDGE(k) \
    do {                     \
    } while (0)
#endif

namespace tcr {

// Level 4 in the last CTA: the G CTA partials, all WARPS warps at once.
// Thread i adds partials i, i + T, i + 2T, ... (T = 32 * WARPS) in index
// order with every load issued before the first add (one L2 round trip),
// then the warp and CTA collapses (D' = 1 x D) as in levels 2-3.  The order
// is fixed by G alone: deterministic.  Returns the total in warp 0.
template <bool kMma, int WARPS>
__device__ __forceinline__ double collapse_partials(const double* partials, int G, double* s_warp) {
    constexpr int T = WARPS * 32;
    constexpr int kPer = 8;  // loads in flight per thread: G <= 8 T (2048) in one round trip
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double a = 0.0;
    for (int base = 0; base < G; base += kPer * T) {
        double v[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int i = base + (int)threadIdx.x + k * T;
            v[k] = (i < G) ? __ldcg(partials + i) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) a += v[k];
    }
    const double wt = warp_collapse<kMma>(a);
    __syncthreads();  // s_warp reuse: every warp has read its level-3 value
    if (lane == 0) s_warp[warp] = wt;
    __syncthreads();
    return warp == 0 ? warp_collapse<kMma>(lane < WARPS ? s_warp[lane] : 0.0) : 0.0;
}

// Levels 2-4.  Every thread of the CTA calls this with its lane value; the
// total lands in out_f32 / out_f64 (device pointers, either may be null).
// With a peer group (pc && pc->nranks > 0) the last CTA then runs the fused
// cross-GPU combine (tcr_peer.cuh) as rank `me` and writes the group total.
template <bool kMma, int WARPS>
__device__ __forceinline__ void complete_block_and_grid(double lane_val, float* out_f32,
                                                        double* out_f64, const DevWorkspace& ws,
                                                        const PeerCombine* pc = nullptr,
                                                        int me = 0) {
    __shared__ double s_warp[WARPS];
    __shared__ unsigned s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double wt = warp_collapse<kMma>(lane_val);
    if (lane == 0) s_warp[warp] = wt;
    TCR_COMPLETE_EDGE(4);
    __syncthreads();
    TCR_COMPLETE_EDGE(5);
    const bool peer = pc && pc->nranks > 0;
    if (gridDim.x == 1) {
        if (warp != 0) return;
        const unsigned long long prev = peer ? peer_counter(*pc, me) : 0ull;
        const double bt = warp_collapse<kMma>(lane < WARPS ? s_warp[lane] : 0.0);
        const double t = peer ? peer_combine(bt, *pc, me, lane, prev) : bt;
        if (lane == 0) {
            if (out_f32) *out_f32 = (float)t;
            if (out_f64) *out_f64 = t;
        }
        return;
    }
    // the peer epoch is loaded before the ticket (off the last CTA's critical path)
    const unsigned long long prev = (peer && warp == 0) ? peer_counter(*pc, me) : 0ull;
    if (warp == 0) {
        const double bt = warp_collapse<kMma>(lane < WARPS ? s_warp[lane] : 0.0);
        TCR_COMPLETE_EDGE(6);
        if (lane == 0) {
            ws.partials[blockIdx.x] = bt;
            TCR_COMPLETE_EDGE(7);
            s_last = (ticket_acq_rel(ws.ticket) == gridDim.x - 1) ? 1u : 0u;
        }
    }
    TCR_COMPLETE_EDGE(8);
    __syncthreads();  // the ticket's acquire, then CTA-wide: all partials visible
    if (!s_last) return;
    double tot = collapse_partials<kMma, WARPS>(ws.partials, (int)gridDim.x, s_warp);
    if (warp != 0) return;
    if (peer) tot = peer_combine(tot, *pc, me, lane, prev);
    if (lane == 0) {
        if (out_f32) *out_f32 = (float)tot;
        if (out_f64) *out_f64 = tot;
        *ws.ticket = 0u;  // self-reset for the next launch on this stream
    }
}

}  // namespace tcr
