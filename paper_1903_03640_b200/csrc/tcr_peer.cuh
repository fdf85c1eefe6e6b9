// tcr_peer.cuh -- NEXT-2: the cross-GPU combine fused into the reduction
// kernel (the paper's "distributed reduction ...
// merged with message passing", §II).
//
// The last CTA of each rank, holding the rank's fp64 partial (level 4 of the
// hierarchy, tcr_complete.cuh), continues instead of exiting.  The epoch of
// the call is the own mailbox's combine counter + 1 -- device-resident, so
// the launch can be captured in a CUDA graph and replayed; every rank makes
// the same sequence of calls, so the counters agree:
//   push  lane d (d != rank) writes the partial into slot [epoch & 1][rank]
//         of rank d's mailbox over NVLink (mapped peer pointer) as ONE
//         16-byte store of two 8-byte words {lo32(value), epoch32},
//         {hi32(value), epoch32};
//   wait  lane r (r != rank) polls slot [epoch & 1][r] of the OWN mailbox
//         until both words carry epoch32 (lane == rank keeps its own value);
//   sum   the P partials in rank order 0..P-1 (fp64), so every rank computes
//         the bitwise identical total, as D' is replicated in Eq. 12.
// Each 8-byte word is written and read single-copy atomically, so a word
// whose flag half matches carries this epoch's data half: no release/acquire
// fence is needed (a .sys-scope fence costs microseconds, measured in
// profiles/r01/peer_emulated.json) -- the flag-in-every-word scheme of
// low-latency collective protocols.
// Two parities make reuse safe without resets: a rank writes parity p again
// (epoch e + 2) only after its epoch-(e + 1) wait saw every peer's e + 1
// words, and a peer posts e + 1 only after its epoch-e kernel (which read
// parity p) finished on its stream.  The wait is bounded by pc.timeout_ns of
// %globaltimer: on expiry the error word of the own mailbox is set and the
// result is NaN, so a missing peer never hangs the GPU.  Consecutive calls of
// one rank are stream-ordered, so the counter needs no atomics.
#pragma once

#include <cstdint>

#include "tcr_internal.h"

namespace tcr {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_slot(void* p, unsigned long long w0, unsigned long long w1) {
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1)
                 : "memory");
}
__device__ __forceinline__ void ld_slot(const void* p, unsigned long long& w0,
                                        unsigned long long& w1) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p)
                 : "memory");
}

struct __align__(16) MailboxSlot {
    unsigned long long w[2];  // {epoch32 << 32 | lo32(partial)}, {epoch32 << 32 | hi32(partial)}
};

__device__ __forceinline__ MailboxSlot* mailbox_slot(void* mbox, unsigned parity, int src) {
    return reinterpret_cast<MailboxSlot*>(mbox) + parity * kMaxPeers + src;
}

// pc.mbox[i] with constant indices only (a dynamic index into a kernel
// parameter array would make the compiler copy the array to local memory).
__device__ __forceinline__ void* mailbox_of(const PeerCombine& pc, int i) {
    void* p = nullptr;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
        if (r == i) p = pc.mbox[r];
    return p;
}

// This rank's combine counter (the previous epoch).  Loaded by warp 0 of
// every CTA before its completion ticket, so that the load's latency is off
// the critical path of whichever CTA turns out to be the last.
__device__ __forceinline__ unsigned long long peer_counter(const PeerCombine& pc, int me) {
    const char* own = static_cast<const char*>(mailbox_of(pc, me));
    return *reinterpret_cast<const volatile unsigned long long*>(own + kMailboxEpochOffset);
}

// Called by all 32 lanes of warp 0 of the rank's last CTA with the rank's
// partial v (every lane's copy equal) and prev = peer_counter(); returns the
// group total in every lane.  `me` is this rank's index in the group.
__device__ __forceinline__ double peer_combine(double v, const PeerCombine& pc, int me, int lane,
                                               unsigned long long prev) {
    const int P = pc.nranks;
    char* own = static_cast<char*>(mailbox_of(pc, me));
    const unsigned long long epoch = prev + 1ull;
    const unsigned par = (unsigned)(epoch & 1ull);
    const unsigned long long tag = (unsigned long long)(unsigned)epoch << 32;
    if (lane < P && lane != me) {  // push: one remote slot per peer (fire and forget)
        const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
        st_slot(mailbox_slot(mailbox_of(pc, lane), par, me), tag | (bits & 0xFFFFFFFFull),
                tag | (bits >> 32));
    }
    double got = v;  // lane == me: the own partial needs no round trip
    unsigned ok = 1u;
    if (lane < P && lane != me) {  // wait for rank `lane`'s partial in the own mailbox
        const MailboxSlot* s = mailbox_slot(own, par, lane);
        unsigned long long w0, w1;
        const unsigned long long t0 = globaltimer_ns();
        for (;;) {
            ld_slot(s, w0, w1);
            if ((w0 >> 32) == (unsigned)epoch && (w1 >> 32) == (unsigned)epoch) break;
            if (globaltimer_ns() - t0 > pc.timeout_ns) {
                ok = 0u;
                break;
            }
            __nanosleep(20);
        }
        got = ok ? __longlong_as_double((long long)((w1 << 32) | (w0 & 0xFFFFFFFFull))) : 0.0;
    }
    const unsigned all_ok = __all_sync(0xffffffffu, ok);
    double tot = 0.0;
    for (int r = 0; r < P; ++r) tot += __shfl_sync(0xffffffffu, got, r);  // rank order
    if (lane == 0) {
        *reinterpret_cast<unsigned long long*>(own + kMailboxEpochOffset) = epoch;
        if (!all_ok) atomicExch(reinterpret_cast<unsigned*>(own + kMailboxErrOffset), 1u);
    }
    if (!all_ok) tot = __longlong_as_double(0x7FF8000000000000ll);  // NaN
    return tot;
}

// ---------------------------------------------------------------------------
// Exact variant (NEXT-2 x NEXT-3): the payload is the rank's int64 limb state
// acc[6] = {l0, l1, l2, n_nan, n_pinf, n_ninf} (tcr_exact.cu), sent as twelve
// 8-byte words {epoch32, one 32-bit half of a limb} in a 96-byte slot of the
// exact region of the mailbox; the sum of the limbs over ranks is exact in
// any order, so every rank finalizes the identical integer.
struct __align__(16) MailboxSlotX {
    unsigned long long w[12];
};

__device__ __forceinline__ MailboxSlotX* mailbox_slot_x(void* mbox, unsigned parity, int src) {
    return reinterpret_cast<MailboxSlotX*>(static_cast<char*>(mbox) + kMailboxExactOffset) +
           parity * kMaxPeers + src;
}

// All 32 lanes of warp 0 of the rank's last CTA, with the rank's limbs in
// every lane; on return every lane holds the group's summed limbs.
__device__ __forceinline__ bool peer_combine_exact(long long (&lim)[6], const PeerCombine& pc,
                                                   int me, int lane, unsigned long long prev) {
    const int P = pc.nranks;
    char* own = static_cast<char*>(mailbox_of(pc, me));
    const unsigned long long epoch = prev + 1ull;
    const unsigned par = (unsigned)(epoch & 1ull);
    const unsigned long long tag = (unsigned long long)(unsigned)epoch << 32;
    if (lane < P && lane != me) {  // push the 12 halves, 16 bytes per store
        MailboxSlotX* d = mailbox_slot_x(mailbox_of(pc, lane), par, me);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const unsigned long long u = (unsigned long long)lim[k];
            st_slot(&d->w[2 * k], tag | (u & 0xFFFFFFFFull), tag | (u >> 32));
        }
    }
    long long got[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) got[k] = lim[k];
    unsigned ok = 1u;
    if (lane < P && lane != me) {
        const MailboxSlotX* src = mailbox_slot_x(own, par, lane);
        unsigned long long w[12];
        const unsigned long long t0 = globaltimer_ns();
        for (;;) {
            bool all = true;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                ld_slot(&src->w[2 * k], w[2 * k], w[2 * k + 1]);
                all = all && (w[2 * k] >> 32) == (unsigned)epoch &&
                      (w[2 * k + 1] >> 32) == (unsigned)epoch;
            }
            if (all) break;
            if (globaltimer_ns() - t0 > pc.timeout_ns) {
                ok = 0u;
                break;
            }
            __nanosleep(20);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k)
            got[k] = ok ? (long long)((w[2 * k + 1] << 32) | (w[2 * k] & 0xFFFFFFFFull)) : 0ll;
    }
    const unsigned all_ok = __all_sync(0xffffffffu, ok);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        long long t = 0;
        for (int r = 0; r < P; ++r) t += __shfl_sync(0xffffffffu, got[k], r);
        lim[k] = t;
    }
    if (lane == 0) {
        *reinterpret_cast<unsigned long long*>(own + kMailboxEpochOffset) = epoch;
        if (!all_ok) atomicExch(reinterpret_cast<unsigned*>(own + kMailboxErrOffset), 1u);
    }
    return all_ok != 0;
}

}  // namespace tcr
