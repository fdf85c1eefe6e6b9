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
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double wt = warp_collapse<kMma>(lane_val);
    if (lane == 0) s_warp[warp] = wt;
    TCR_COMPLETE_EDGE(4);
    __syncthreads();
    TCR_COMPLETE_EDGE(5);
    if (warp != 0) return;
    const bool peer = pc && pc->nranks > 0;
    const unsigned long long prev = peer ? peer_counter(*pc, me) : 0ull;
    const double bt = warp_collapse<kMma>(lane < WARPS ? s_warp[lane] : 0.0);
    if (gridDim.x == 1) {
        const double t = peer ? peer_combine(bt, *pc, me, lane, prev) : bt;
        if (lane == 0) {
            if (out_f32) *out_f32 = (float)t;
            if (out_f64) *out_f64 = t;
        }
        return;
    }
    unsigned last = 0;
    TCR_COMPLETE_EDGE(6);
    if (lane == 0) {
        ws.partials[blockIdx.x] = bt;
        __threadfence();  // release the partial before taking a ticket
        TCR_COMPLETE_EDGE(7);
        last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
    TCR_COMPLETE_EDGE(8);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();  // acquire: every other CTA's partial is visible
    double v = 0.0;
    for (int i = lane; i < (int)gridDim.x; i += 32) v += __ldcg(ws.partials + i);  // fixed order
    double tot = warp_collapse<kMma>(v);
    if (peer) tot = peer_combine(tot, *pc, me, lane, prev);
    if (lane == 0) {
        if (out_f32) *out_f32 = (float)tot;
        if (out_f64) *out_f64 = tot;
        *ws.ticket = 0u;  // self-reset for the next launch on this stream
    }
}

}  // namespace tcr
