// tcr_tcgen05.cu -- the Blackwell-native MMA-encoded reduction:
//
//   HBM --(bulk async copy, TMA engine)--> SMEM ring --(tcgen05.mma, A from
//   SMEM, B = all-ones in SMEM)--> fp32 accumulator in TMEM --(tcgen05.ld of
//   one column per accumulator, once per round)--> fp64 registers -> 1 x D.
//
// The input never passes through registers: the tensor core reads each
// 4 KiB chunk of X straight from shared memory as a 128x16 A tile.  Any
// bijection of the chunk onto the tile is a valid placement of the group
// (permutation invariance, reading G1); the no-swizzle K-major descriptor
// below (LBO = 128 B, SBO = 256 B) tiles the 4 KiB contiguously.
//
// Paper mapping (arXiv 1903.03640):
//   D = A x 1 + C (Eq. 9-10): tcgen05.mma M=128, N=16, K=16,
//     B = ones.  Every column of D holds the 128 row sums (Eq. 10);
//     C is carried over the K = stage_bytes / 4 KiB tiles of one chunk
//     (enable_input_d), then the chunk's accumulator slot is read out.
//   D' = 1 x D (Eq. 11-12): fp64 DMMA collapse of the row sums
//     (warp), of the warps (CTA) and of the CTAs (grid, last-CTA ticket).
//
// Warp roles (192 threads, 1 CTA per SM):
//   warp 0   lane 0: producer -- bulk copies into the SMEM ring
//   warp 1   lane 0: MMA issuer; the whole warp allocates TMEM
//   warps 2-5      : epilogue -- drain TMEM slots into fp64, ragged edges
#include <map>
#include <mutex>

#ifdef TCR_TC05_TRACE
namespace tcr {
__device__ unsigned long long g_tc05_edges[10][2048];
}
#define TCR_COMPLETE_EDGE(k)                                                               \
    do {                                                                                   \
        if (threadIdx.x == 0 && blockIdx.x < 2048) {                                       \
            unsigned long long t_;                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
            tcr::g_tc05_edges[k][blockIdx.x] = t_;                                         \
        }                                                                                  \
    } while (0)
#endif
#include "tcr_complete.cuh"
#include "tcr_device.cuh"
#include "tcr_int128.cuh"
#include "tcr_internal.h"
#include "tcr_sm100.cuh"

namespace tcr {

#ifdef TCR_TC05_TRACE
// Diagnostic timeline of CTA 0 (scripts/tc05_trace.cu compiles this file with
// -DTCR_TC05_TRACE): [0] producer issues chunk i, [1] MMA thread sees chunk i
// full, [2] MMA thread committed chunk i, [3] epilogue sees round r full.
__device__ unsigned long long g_tc05_trace[6][4096];  // [4] each MMA issued, [5] tempty seen
__device__ __forceinline__ unsigned long long tc05_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TC05_TRACE(role, idx)                                                    \
    do {                                                                         \
        if (blockIdx.x == 0 && (idx) < 4096) g_tc05_trace[role][idx] = tc05_now(); \
    } while (0)
// per-CTA phase edges: [0] entry, [1] setup done, [2] data phase done,
// [3] exit, [4..8] inside complete_block_and_grid (TCR_COMPLETE_EDGE)
#define TC05_EDGE(k) TCR_COMPLETE_EDGE(k)
#else
#define TC05_EDGE(k) \
    do {             \
    } while (0)
#define TC05_TRACE(role, idx) \
    do {                      \
    } while (0)
#endif

namespace {

constexpr int kTcWarps = 6;
constexpr uint32_t kSlotCols = 16;                   // N = 16 fp32 columns per accumulator
constexpr uint32_t kTileBytes = 128 * 16 * 2;        // one 128x16 fp16 A tile = 4 KiB
constexpr uint32_t kHeaderBytes = 1024;              // ones tile + barriers + TMEM address
constexpr uint32_t kIdesc = sm100::idesc_f16_f32(128, 16);

}  // namespace

struct Tc05Params {
    int stages;            // SMEM ring stages
    uint32_t stage_bytes;  // bytes per stage (multiple of 4 KiB)
    int slots;             // independent accumulators per TMEM buffer (power of 2, <= 16)
    int chain;             // MMAs carried per accumulator before its flush (K)
    int prefetch;          // L2 prefetch distance in chunks (0 = off)
    int split;             // bulk copies per stage
    int interleave;        // 0: CTA b owns a contiguous run of chunks; 1: chunks b, b+G, b+2G, ...
    int dynamic;           // kDyn: percent of the chunks handed out from ws.chunk_next
    uint32_t idesc;        // instruction descriptor (kind::f16 with F16 or BF16 operands)
    uint32_t one_bits;     // 1.0 in the input type (the all-ones B)
    int fmt;               // element format (0 f16, 1 bf16, 2 e4m3, 3 e5m2)
    long long* out_acc;    // kDyn, exact E4M3 entry: the 6-word exact state (else null)
};

// Levels 3-4 of the dynamic-tail variant (kDyn).  Only lane 0 of each
// epilogue warp holds a value (its exact integer T in units of 2^-24 and the
// sum `sp` of the non-finite level-2 totals it saw; the last CTA's ragged
// work is folded into its warp's lane 0 before the call) and has written it
// to s_part[warp] before the CTA barrier that ends the roles.  Thread 0 adds
// the CTA's entries, stores the 3-word CTA partial and takes the ticket; the
// last CTA then loads all G partials at once (one per thread: one L2 round
// trip), adds them as integers (order-free), rounds T * 2^-24 once (RNE) --
// or returns sp when some total was inf / NaN (inf + -inf = NaN in any
// order) -- and resets the ticket and the chunk counter for the next launch
// on this stream.
struct UnitsPart {
    long long lo, hi, sp;  // T = hi:lo, sp as binary64 bits
};

// out_acc (the exact E4M3 entry, r02 §16): the exact state {l0, l1, l2,
// n_nan, n_pinf, n_ninf} of T with l0, l1 in [0, 2^40); when a level-2 total
// was NaN the limbs are 0 and acc[4] = -1 asks rows_nan_fixup_kernel for the
// NaN count (E4M3 has no infinities).
template <int WARPS>
__device__ __forceinline__ void complete_units_grid(const UnitsPart* s_part, float* out_f32,
                                                    double* out_f64, const DevWorkspace& ws,
                                                    const PeerCombine* pc, int me,
                                                    long long* out_acc = nullptr) {
    constexpr int kThreads = WARPS * 32;
    __shared__ UnitsPart s_red[WARPS];
    __shared__ unsigned s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool peer = pc && pc->nranks > 0;
    const unsigned long long prev = (peer && warp == 0) ? peer_counter(*pc, me) : 0ull;
    long long* parts = reinterpret_cast<long long*>(ws.partials);  // 3 words per CTA
    TCR_COMPLETE_EDGE(4);
    TCR_COMPLETE_EDGE(5);
    if (threadIdx.x == 0) {
        i128 b = 0;
        double q = 0.0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            b += make_i128(s_part[w].lo, s_part[w].hi);
            q += __longlong_as_double(s_part[w].sp);
        }
        TCR_COMPLETE_EDGE(6);
        if (gridDim.x > 1) {
            long long* p = parts + 3 * (size_t)blockIdx.x;
            p[0] = (long long)(unsigned long long)b;
            p[1] = (long long)(b >> 64);
            p[2] = __double_as_longlong(q);
            TCR_COMPLETE_EDGE(7);
            if (peer) {
                __threadfence();
                s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
            } else {
                s_last = (ticket_acq_rel(ws.ticket) == gridDim.x - 1) ? 1u : 0u;
            }
        } else {
            s_last = 1u;
            s_red[0] = UnitsPart{(long long)(unsigned long long)b, (long long)(b >> 64),
                                 __double_as_longlong(q)};
        }
    }
    TCR_COMPLETE_EDGE(8);
    __syncthreads();  // thread 0's acquire, then CTA-wide: every partial visible
    TCR_COMPLETE_EDGE(9);
    if (!s_last) return;
    if (gridDim.x > 1) {
        if (peer) __threadfence();
        i128 b = 0;
        double q = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) {
            const long long* p = parts + 3 * (size_t)i;
            b += make_i128(__ldcg(p), __ldcg(p + 1));
            q += __longlong_as_double(__ldcg(p + 2));
        }
        b = warp_sum_i128(b);
        q = warp_collapse_shfl(q);
        if (lane == 0) s_red[warp] = UnitsPart{(long long)(unsigned long long)b, (long long)(b >> 64),
                                                __double_as_longlong(q)};
        __syncthreads();
    }
    if (warp != 0) return;
    i128 b = 0;  // warp 0, every lane the same sums (peer_combine needs the warp)
    double q = 0.0;
    const int nred = gridDim.x > 1 ? WARPS : 1;
    for (int w = 0; w < nred; ++w) {
        b += make_i128(s_red[w].lo, s_red[w].hi);
        q += __longlong_as_double(s_red[w].sp);
    }
    if (lane == 0) {
        if (gridDim.x > 1) *ws.ticket = 0u;
        *ws.chunk_next = 0u;  // every CTA's chunk tickets precede its completion ticket
    }
    float f;
    double d;
    if (q != 0.0) {  // some level-2 total was inf or NaN
        f = (float)q;
        d = q;
    } else {
        round_units_f32_f64(b, f, d);
    }
    if (peer) {
        d = peer_combine(d, *pc, me, lane, prev);
        f = (float)d;
    }
    if (lane == 0) {
        if (out_f32) *out_f32 = f;
        if (out_f64) *out_f64 = d;
        if (out_acc) {
            const bool spc = q != 0.0;
            const u128 m40 = ((u128)1 << 40) - 1;
            out_acc[0] = spc ? 0 : (long long)((u128)b & m40);
            out_acc[1] = spc ? 0 : (long long)(((u128)b >> 40) & m40);
            out_acc[2] = spc ? 0 : (long long)(b >> 80);
            out_acc[3] = 0;
            out_acc[4] = spc ? -1 : 0;
            out_acc[5] = 0;
        }
    }
}

// Accumulator schedule: MMA number j of this CTA (j = 0, 1, ...) goes to
// round r = j / (slots*chain), slot j % slots of TMEM buffer r & 1, and
// accumulates unless it is the slot's first MMA of the round.  Consecutive
// MMAs therefore target different accumulators (no read-after-write chain
// between neighbours), each accumulator carries `chain` tiles (bounded
// truncation, reading G10), and the epilogue drains one buffer per round
// while the tensor core fills the other.
// KM > 0 (r02): one accumulator round per SMEM stage -- KM MMAs per stage
// over 4 accumulators (chain KM / 4) -- and a tight, fully unrolled issue
// loop: the issuing thread waits full[s] and tempty[buf] once per stage, issues
// the KM MMAs with compile-time descriptor / TMEM offsets and commits twice.
// The generic loop (KM = 0) spent ~190 ns of issuing-thread time per MMA on
// its per-MMA bookkeeping (scripts/tc05_trace.cu: MMA issue gap, r02), against
// ~37 ns for a bare issue loop (scripts/tc05_floor.cu) -- which is why r01
// needed three CTAs (three issuers) per SM.
// kPeer: the NEXT-2 variant (the cross-GPU combine fused into the last CTA,
// tcr_peer.cuh), as for the streaming kernel; grid.y slices = emulated ranks.
// kDyn (r02 §16): the dynamic tail.  CTA b first streams its contiguous run
// of the first (100 - dynamic) % of the chunks, then takes the remaining
// chunks one at a time from ws.chunk_next (the producer holds two tickets
// ahead, so the atomic's latency overlaps the ring), so every SM stops
// within about one chunk of the others instead of waiting for the slowest
// static run.  The producer marks each ring stage valid or END; the MMA
// issuer forwards END to the epilogue through a per-buffer flag.  Order-free
// arithmetic keeps the result independent of the schedule: each round's
// 4 x 128 fp32 row sums (multiples of 2^-24, as every binary16 / fp8 value
// and every fp32 sum of them is) are collapsed per warp by the DMMA D' = 1 x D
// (exact: |total| < 2^29, i.e. < 2^53 units) and added as integers.
template <bool kF8, int KM, bool kPeer = false, bool kDyn = false>
__global__ void __launch_bounds__(kTcWarps * 32)
reduce_tcgen05_kernel(const uint8_t* __restrict__ x, size_t n, Tc05Params prm, float* out_f32,
                      double* out_f64, DevWorkspace ws, PeerCombine pc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    TC05_EDGE(0);
    int me = pc.rank;
    if (kPeer && gridDim.y > 1) {  // emulated peer group: slice y is rank y, reducing its shard
        const size_t P = gridDim.y, r = blockIdx.y, es = prm.fmt >= 2 ? 1u : 2u;
        const size_t lo = r * n / P, hi = (r + 1) * n / P;
        x += lo * es;
        n = hi - lo;
        ws.partials += (kDyn ? 3 : 1) * r * gridDim.x;  // kDyn: 3 words per CTA partial
        ws.ticket += r;
        ws.chunk_next += r;
        if (out_f32) out_f32 += r;
        if (out_f64) out_f64 += r;
        me = (int)r;
    }
    static_assert(!kDyn || KM > 0, "the dynamic tail runs the tight issue loop");
    // exactness of the per-round DMMA collapse: 32 lanes x 4 slots x (KM / 4)
    // MMAs x K elements x the largest magnitude < 2^29 (binary16: K = 16,
    // 65504; fp8: K = 32, 57344 for E5M2 -- so fp8 takes KM <= 8)
    static_assert(!kDyn || (kF8 ? 32.0 * KM * 32 * 57344.0 : 32.0 * KM * 16 * 65504.0) < 536870912.0,
                  "per-round collapse must stay below 2^53 units");
    const int stages = prm.stages;
    const uint32_t stage_bytes = prm.stage_bytes;
    const uint32_t buf_cols = (uint32_t)prm.slots * kSlotCols;
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem);             // 512 B of ones (B operand)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 512);       // [stages]
    uint64_t* empty = full + stages;                                // [stages]
    uint64_t* tfull = empty + stages;                               // [2]
    uint64_t* tempty = tfull + 2;                                   // [2]
    volatile uint32_t* sinfo = reinterpret_cast<volatile uint32_t*>(tempty + 2);  // [stages] kDyn
    volatile uint32_t* tend = sinfo + stages;                                       // [2] kDyn
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kHeaderBytes - 8);
    uint8_t* ring = smem + kHeaderBytes;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // all index math in bytes (n elements of 1 or 2 bytes)
    const size_t nbytes = n * (prm.fmt >= 2 ? 1u : 2u);
    size_t head = (16u - ((uintptr_t)x & 15u)) & 15u;
    if (head > nbytes) head = nbytes;
    const uint8_t* xa = x + head;
    const size_t nb = nbytes - head;
    const size_t C = nb / stage_bytes;
    const size_t G = gridDim.x, b = blockIdx.x;
    // kDyn: chunks [0, Cs) statically (contiguous runs), [Cs, C) by ticket
    const size_t D = kDyn ? C * (size_t)prm.dynamic / 100u : 0;
    const size_t Cs = C - D;
    const size_t c_begin = kDyn ? b * Cs / G : prm.interleave ? b : b * C / G;
    const int nchunks = kDyn ? (int)((b + 1) * Cs / G - b * Cs / G)
                        : prm.interleave ? (int)(C > b ? (C - b + G - 1) / G : 0)
                                         : (int)((b + 1) * C / G - b * C / G);
    const size_t chunk_step = (!kDyn && prm.interleave) ? G * (size_t)stage_bytes : (size_t)stage_bytes;
    const int kmma = (int)(stage_bytes / kTileBytes);
    const int per_round = prm.slots * prm.chain;
    const long long total_mma = (long long)nchunks * kmma;

    // The producer (thread 0) initialises the barriers and issues the first
    // ring's worth of bulk copies right away (r02): their HBM latency then
    // overlaps the rest of the set-up (ones tile, TMEM allocation, the CTA
    // barrier) instead of following it.  It waits for the previous kernel
    // (PDL) before touching x; the other threads do after the CTA barrier.
    const uint64_t pol = sm100::policy_evict_first();
    const uint32_t piece = stage_bytes / (uint32_t)prm.split;
    const int pre = nchunks < stages ? nchunks : stages;  // chunks issued before the barrier
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            sm100::mbar_init(&tfull[b], 1);
            sm100::mbar_init(&tempty[b], 4);
            if (kDyn) tend[b] = 0u;
        }
        sm100::fence_mbar_init();
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint8_t* src = xa + c_begin * (size_t)stage_bytes;
        for (int i = 0; i < pre; ++i, src += chunk_step) {  // ring stage i, first phase: free
            TC05_TRACE(0, i);
            if (kDyn) sinfo[i] = 1u;
            sm100::mbar_arrive_expect_tx(&full[i], stage_bytes);
            uint8_t* dst = ring + (size_t)i * stage_bytes;
            for (int q = 0; q < prm.split; ++q)
                sm100::bulk_g2s(dst + (size_t)q * piece, src + (size_t)q * piece, piece, &full[i], pol);
        }
    }
    for (int i = threadIdx.x; i < 128; i += blockDim.x) ones[i] = prm.one_bits;
    sm100::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
    const uint32_t tmem_cols = 2u * buf_cols < 32u ? 32u : 2u * buf_cols;
    if (warp == 1) sm100::tmem_alloc(tmem_slot, tmem_cols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    TC05_EDGE(1);
    // PDL: the CTA-local set-up above (barriers, ones tile, TMEM) overlaps the
    // previous kernel's tail; nothing global is touched before this wait
    pdl_wait_and_release();

    double acc = 0.0;
    i128 T = 0;       // kDyn: exact sum in units of 2^-24
    double sp = 0.0;  // kDyn: sum of the non-finite level-2 totals
    if constexpr (kDyn) {
        if (warp == 0) {
            if (lane == 0) {  // producer: static run, then chunk tickets, then END
                int s = pre % stages;
                uint32_t ph = (uint32_t)(pre / stages);
                auto issue = [&](const uint8_t* src) {
                    sm100::mbar_wait(&empty[s], ph ^ 1u);
                    sinfo[s] = 1u;
                    sm100::mbar_arrive_expect_tx(&full[s], stage_bytes);
                    uint8_t* dst = ring + (size_t)s * stage_bytes;
                    for (int q = 0; q < prm.split; ++q)
                        sm100::bulk_g2s(dst + (size_t)q * piece, src + (size_t)q * piece, piece, &full[s], pol);
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                };
                // two tickets held ahead: each is fetched about two chunks before
                // it is needed (its result is first read by the `t >= D` test)
                unsigned t0 = 0u, t1 = 0u;
                bool f0 = false, f1 = false;
                const uint8_t* src = xa + (c_begin + (size_t)pre) * (size_t)stage_bytes;
                for (int i = pre; i < nchunks; ++i, src += stage_bytes) {
                    if (D && !f0 && nchunks - i <= 2) {
                        t0 = atomicAdd(ws.chunk_next, 1u);
                        f0 = true;
                    }
                    if (D && !f1 && nchunks - i <= 1) {
                        t1 = atomicAdd(ws.chunk_next, 1u);
                        f1 = true;
                    }
                    issue(src);
                }
                if (D) {
                    if (!f0) t0 = atomicAdd(ws.chunk_next, 1u);
                    if (!f1) t1 = atomicAdd(ws.chunk_next, 1u);
                    for (;;) {
                        const unsigned t = t0;
                        t0 = t1;
                        t1 = atomicAdd(ws.chunk_next, 1u);
                        if ((size_t)t >= D) break;
                        issue(xa + (Cs + (size_t)t) * (size_t)stage_bytes);
                    }
                }
                sm100::mbar_wait(&empty[s], ph ^ 1u);  // END: a stage with no bytes
                sinfo[s] = 0u;
                sm100::mbar_arrive(&full[s]);
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0) {  // MMA issuer: one round per valid stage, then END to the epilogue
                const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
                const uint64_t adesc0 = sm100::smem_desc_kmajor(sm100::smem_addr(ring), 128, 256);
                const uint64_t stage_step = stage_bytes >> 4;
                constexpr uint64_t kTileStep = kTileBytes >> 4;
                int s = 0, buf = 0;
                uint32_t ph = 0, use = 0;
                for (;;) {
                    sm100::mbar_wait(&full[s], ph);
                    if (sinfo[s] == 0u) break;
                    sm100::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);  // drained two rounds ago
                    sm100::tc_fence_after();
                    const uint64_t a = adesc0 + (uint64_t)s * stage_step;
                    const uint32_t d = tmem + (uint32_t)buf * (4u * kSlotCols);
    #pragma unroll
                    for (int k = 0; k < (KM > 0 ? KM : 1); ++k) {
                        if constexpr (kF8)
                            sm100::mma_f8_ss(d + (uint32_t)(k & 3) * kSlotCols, a + (uint64_t)k * kTileStep,
                                             bdesc, prm.idesc, k >= 4 ? 1u : 0u);
                        else
                            sm100::mma_f16_ss(d + (uint32_t)(k & 3) * kSlotCols, a + (uint64_t)k * kTileStep,
                                              bdesc, prm.idesc, k >= 4 ? 1u : 0u);
                    }
                    sm100::mma_commit(&tfull[buf]);
                    sm100::mma_commit(&empty[s]);
                    if (buf) ++use;
                    buf ^= 1;
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                sm100::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);  // that buffer's last round drained
                tend[buf] = 1u;
                sm100::mbar_arrive(&tfull[buf]);
            }
            __syncwarp();
        } else {  // epilogue warps 2..5: one round per valid stage until END
            const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
            int buf = 0;
            uint32_t use = 0;
            for (;;) {
                sm100::mbar_wait(&tfull[buf], use & 1u);
                if (tend[buf]) break;
                sm100::tc_fence_after();
                const uint32_t base = tmem + (quarter << 16) + (uint32_t)buf * (4u * kSlotCols);
                uint32_t v[4];
    #pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = sm100::tmem_ld_32x32b_x1(base + (uint32_t)q * kSlotCols);
                sm100::tmem_wait_ld();
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[buf]);
                if (buf) ++use;
                buf ^= 1;
                // level 2: D' = 1 x D over the warp's 32 rows x 4 accumulators (exact)
                const double w = ((double)__uint_as_float(v[0]) + (double)__uint_as_float(v[1])) +
                                 ((double)__uint_as_float(v[2]) + (double)__uint_as_float(v[3]));
                const double tot = warp_collapse<true>(w);
                if (lane == 0) {
                    if (isfinite(tot)) T += (i128)__double2ll_rn(tot * 0x1p24);
                    else sp += tot;
                }
            }
            if (blockIdx.x == gridDim.x - 1) {
                // ragged work (< one chunk past the last full chunk, and the
                // unaligned head): 512-byte mma.sync tiles, zero padded; a lane's
                // rows stay below 2^27 (< 2^51 units): exact in binary64
                const int e = warp - 2;
                const uint8_t* xr = xa + C * (size_t)stage_bytes;
                const size_t rem = nb - C * (size_t)stage_bytes;
                const size_t Tr = rem / 512;
                const int tail = (int)(rem - Tr * 512);
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                double racc = 0.0;
                const uint4* base = reinterpret_cast<const uint4*>(xr) + lane;
                auto tile = [&](const uint4& v) {
                    switch (prm.fmt) {
                        case 2: mma_rowsum_fp8_as_f16<kE4M3>(c, v); break;
                        case 3: mma_rowsum_fp8_as_f16<kE5M2>(c, v); break;
                        default: mma_rowsum(c, v); break;
                    }
                    flush_rows(c, racc, lane);
                };
                for (size_t t = e; t < Tr; t += 4) tile(ldg_stream(base + t * 32));
                if (e == 0 && head) tile(load_ragged_bytes(x, (int)head, lane));
                if (e == 1 && tail) tile(load_ragged_bytes(xr + Tr * 512, tail, lane));
                // into lane 0 (every lane's rows: exact integers below 2^51; the
                // warp's sum below 2^56)
                long long u = 0;
                double spl = 0.0;
                if (isfinite(racc)) u = __double2ll_rn(racc * 0x1p24);
                else spl = racc;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    u += __shfl_xor_sync(0xffffffffu, u, o);
                    spl += __shfl_xor_sync(0xffffffffu, spl, o);
                }
                if (lane == 0) {
                    T += (i128)u;
                    sp += spl;
                }
            }
        }
    } else {
        if (warp == 0) {
            if (lane == 0 && nchunks > pre) {  // producer: the chunks after the first ring
                const uint8_t* src = xa + c_begin * (size_t)stage_bytes + (size_t)pre * chunk_step;
                for (int i = pre; i < pre + prm.prefetch && i < nchunks; ++i)
                    sm100::prefetch_l2(src + (size_t)(i - pre) * chunk_step, stage_bytes);
                int s = pre % stages;
                uint32_t ph = pre / stages;  // pre <= stages: the first ring is one phase
                for (int i = pre; i < nchunks; ++i, src += chunk_step) {
                    if (prm.prefetch && i + prm.prefetch < nchunks)
                        sm100::prefetch_l2(src + (size_t)prm.prefetch * chunk_step, stage_bytes);
                    sm100::mbar_wait(&empty[s], ph ^ 1u);
                    TC05_TRACE(0, i);
                    sm100::mbar_arrive_expect_tx(&full[s], stage_bytes);
                    uint8_t* dst = ring + (size_t)s * stage_bytes;
                    for (int q = 0; q < prm.split; ++q)
                        sm100::bulk_g2s(dst + (size_t)q * piece, src + (size_t)q * piece, piece, &full[s],
                                        pol);
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            __syncwarp();
        } else if (KM > 0 && warp == 1) {
            if (lane == 0 && nchunks > 0) {  // MMA issuer, one round per stage (tight loop)
                const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
                const uint64_t adesc0 = sm100::smem_desc_kmajor(sm100::smem_addr(ring), 128, 256);
                const uint64_t stage_step = stage_bytes >> 4;
                constexpr uint64_t kTileStep = kTileBytes >> 4;
                int s = 0, buf = 0;
                uint32_t ph = 0, use = 0;
                for (int i = 0; i < nchunks; ++i) {
                    sm100::mbar_wait(&full[s], ph);
                    sm100::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);  // drained two rounds ago
                    TC05_TRACE(1, i);
                    sm100::tc_fence_after();
                    const uint64_t a = adesc0 + (uint64_t)s * stage_step;
                    const uint32_t d = tmem + (uint32_t)buf * (4u * kSlotCols);
    #pragma unroll
                    for (int k = 0; k < (KM > 0 ? KM : 1); ++k) {
                        if constexpr (kF8)
                            sm100::mma_f8_ss(d + (uint32_t)(k & 3) * kSlotCols, a + (uint64_t)k * kTileStep,
                                             bdesc, prm.idesc, k >= 4 ? 1u : 0u);
                        else
                            sm100::mma_f16_ss(d + (uint32_t)(k & 3) * kSlotCols, a + (uint64_t)k * kTileStep,
                                              bdesc, prm.idesc, k >= 4 ? 1u : 0u);
                    }
                    sm100::mma_commit(&tfull[buf]);  // this round's accumulators, once complete
                    sm100::mma_commit(&empty[s]);    // SMEM stage free once these MMAs complete
                    TC05_TRACE(2, i);
                    if (buf) ++use;
                    buf ^= 1;
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            if (lane == 0 && nchunks > 0) {  // MMA issuer
                const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
                const uint64_t adesc0 = sm100::smem_desc_kmajor(sm100::smem_addr(ring), 128, 256);
                const uint64_t stage_step = stage_bytes >> 4, tile_step = kTileBytes >> 4;
                const uint32_t last_slot = (uint32_t)prm.slots - 1;
                int s = 0;
                uint32_t ph = 0;
                int pos = 0;          // MMA index within the current round
                int buf = 0;          // TMEM buffer of the current round
                uint32_t use = 0;     // how many times `buf` was filled before (parity)
                long long left = total_mma;
                for (int i = 0; i < nchunks; ++i) {
                    sm100::mbar_wait(&full[s], ph);
                    TC05_TRACE(1, i);
                    sm100::tc_fence_after();
                    uint64_t adesc = adesc0 + (uint64_t)s * stage_step;
                    for (int k = 0; k < kmma; ++k, adesc += tile_step) {
                        if (pos == 0) {  // buffer drained by the epilogue two rounds ago?
                            sm100::mbar_wait(&tempty[buf], (use & 1u) ^ 1u);
                            sm100::tc_fence_after();
                            TC05_TRACE(5, (int)((total_mma - left) / per_round));
                        }
                        const uint32_t d = tmem + (uint32_t)buf * buf_cols +
                                           ((uint32_t)pos & last_slot) * kSlotCols;
                        if constexpr (kF8)
                            sm100::mma_f8_ss(d, adesc, bdesc, prm.idesc, pos >= prm.slots ? 1u : 0u);
                        else
                            sm100::mma_f16_ss(d, adesc, bdesc, prm.idesc, pos >= prm.slots ? 1u : 0u);
                        TC05_TRACE(4, (int)(total_mma - left));
                        --left;
                        if (++pos == per_round || left == 0) {
                            sm100::mma_commit(&tfull[buf]);
                            pos = 0;
                            if (buf) ++use;
                            buf ^= 1;
                        }
                    }
                    sm100::mma_commit(&empty[s]);  // SMEM stage free once these MMAs complete
                    TC05_TRACE(2, i);
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            }
            __syncwarp();
        } else {  // epilogue warps 2..5: TMEM lane quarter (warp % 4)
            const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
            const long long rounds = (total_mma + per_round - 1) / per_round;
            long long left = total_mma;
            int buf = 0;
            uint32_t use = 0;
            for (long long r = 0; r < rounds; ++r) {
                const int valid = left < prm.slots ? (int)left : prm.slots;
                left -= per_round;
                sm100::mbar_wait(&tfull[buf], use & 1u);
                if (lane == 0 && warp == 2) TC05_TRACE(3, (int)r);
                sm100::tc_fence_after();
                const uint32_t base = tmem + (quarter << 16) + (uint32_t)buf * buf_cols;
                for (int s0 = 0; s0 < valid; s0 += 4) {
                    uint32_t v[4];
    #pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (s0 + q < valid)
                            v[q] = sm100::tmem_ld_32x32b_x1(base + (uint32_t)(s0 + q) * kSlotCols);
                    sm100::tmem_wait_ld();
    #pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (s0 + q < valid) acc += (double)__uint_as_float(v[q]);
                }
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[buf]);
                if (buf) ++use;
                buf ^= 1;
            }
            if (blockIdx.x == gridDim.x - 1) {
                // Ragged work (< one chunk past the last full chunk, and the
                // unaligned head): 512-byte mma.sync tiles, zero padded.
                const int e = warp - 2;
                const uint8_t* xr = xa + C * (size_t)stage_bytes;
                const size_t rem = nb - C * (size_t)stage_bytes;
                const size_t Tr = rem / 512;
                const int tail = (int)(rem - Tr * 512);
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                const uint4* base = reinterpret_cast<const uint4*>(xr) + lane;
                auto tile = [&](const uint4& v) {
                    switch (prm.fmt) {
                        case 1: mma_rowsum_bf16(c, v); break;
                        case 2: mma_rowsum_fp8_as_f16<kE4M3>(c, v); break;
                        case 3: mma_rowsum_fp8_as_f16<kE5M2>(c, v); break;
                        default: mma_rowsum(c, v); break;
                    }
                    flush_rows(c, acc, lane);
                };
                for (size_t t = e; t < Tr; t += 4) tile(ldg_stream(base + t * 32));
                if (e == 0 && head) tile(load_ragged_bytes(x, (int)head, lane));
                if (e == 1 && tail) tile(load_ragged_bytes(xr + Tr * 512, tail, lane));
            }
        }
    }
    __shared__ UnitsPart s_units[kTcWarps];  // kDyn: lane 0 of every warp (zero for warps 0, 1)
    if (kDyn && lane == 0)
        s_units[warp] = UnitsPart{(long long)(unsigned long long)T, (long long)(T >> 64),
                                  __double_as_longlong(sp)};
    sm100::tc_fence_before();
    __syncthreads();
    TC05_EDGE(2);
    if (warp == 1) sm100::tmem_dealloc(tmem, tmem_cols);
    if constexpr (kDyn)
        complete_units_grid<kTcWarps>(s_units, out_f32, out_f64, ws, kPeer ? &pc : nullptr, me, prm.out_acc);
    else
        complete_block_and_grid<true, kTcWarps>(acc, out_f32, out_f64, ws, kPeer ? &pc : nullptr, me);
    TC05_EDGE(3);
}

// CTAs of this kernel that can be co-resident on one SM for `cfg`: the
// requested count, clamped by shared memory (227 KiB per SM) and by TMEM
// (512 columns per SM; each CTA allocates 2 buffers x slots x 16 columns).
static int tc05_resident(const LaunchCfg& cfg) {
    const size_t smem = kHeaderBytes + (size_t)cfg.tc05_stages * (size_t)cfg.tc05_stage_kb * 1024u;
    const int tmem_cols = 2 * cfg.tc05_slots * (int)kSlotCols < 32 ? 32 : 2 * cfg.tc05_slots * (int)kSlotCols;
    int r = cfg.tc05_ctas < 1 ? 1 : cfg.tc05_ctas;
    const int by_smem = (int)((227u * 1024u) / smem);
    const int by_tmem = 512 / tmem_cols;
    if (r > by_smem) r = by_smem;
    if (r > by_tmem) r = by_tmem;
    return r < 1 ? 1 : r;
}

int tcgen05_grid(size_t nbytes, const LaunchCfg& cfg) {
    const size_t C = nbytes / ((size_t)cfg.tc05_stage_kb * 1024);
    const size_t gmax = (size_t)cfg.sms * (size_t)tc05_resident(cfg);
    size_t g = C < gmax ? C : gmax;
    return g < 1 ? 1 : (int)g;
}

// TCR_CFG_TC05_CTAS_PER_SM = 0 (auto, the default since r02): one CTA (one
// issuer) per SM with the configured ring from 256 MiB of input, where the
// tight issue loop keeps up with HBM alone; below, several CTAs per SM with
// short rings, so that a short input is spread over more independent
// pipelines.  With the library's default ring (4 x 32 KiB, 4 accumulators x
// chain 2) the shape below 256 MiB follows the measured best per size
// (profiles/r02/tc05_small_sweep3.txt, warm CUDA graphs, time / mma.sync's):
// 16 MiB and 64 MiB 3 x 32 KiB at 2 CTAs (1.21, 1.12), 32 MiB 2 x 16 KiB at
// 3 CTAs (1.22), otherwise 2 x 32 KiB at 3 CTAs (1.07-1.25).
static LaunchCfg tc05_effective(size_t nbytes, const LaunchCfg& cfg) {
    LaunchCfg c = cfg;
    if (c.tc05_ctas == 0) {
        const bool default_ring = c.tc05_stages == 4 && c.tc05_stage_kb == 32 && c.tc05_slots == 4 &&
                                  c.tc05_chain == 2;
        const size_t mib = nbytes >> 20;
        if (nbytes >= ((size_t)256 << 20)) {
            c.tc05_ctas = 1;
        } else if (default_ring && ((mib >= 12 && mib < 24) || (mib >= 48 && mib < 96))) {
            c.tc05_ctas = 2;
            c.tc05_stages = 3;
        } else if (default_ring && mib >= 24 && mib < 48) {
            c.tc05_ctas = 3;
            c.tc05_stages = 2;
            c.tc05_stage_kb = 16;
            c.tc05_chain = 1;
        } else {
            c.tc05_ctas = 3;
            if (c.tc05_stages > 2) c.tc05_stages = 2;
        }
    }
    return c;
}

using Tc05Kernel = void (*)(const uint8_t*, size_t, Tc05Params, float*, double*, DevWorkspace,
                           PeerCombine);

// The instantiation for (format, MMAs per stage): the tight issue loop for
// KM = 4, 8, 16 (the peer variant: 8, the default, else the generic loop).
// dyn: the dynamic-tail variant (binary16 / fp8 with the tight loop; fp8 up
// to 8 MMAs per stage, the exactness bound of the per-round collapse).
template <bool kPeer>
static Tc05Kernel tc05_kernel(bool f8, int km, bool dyn) {
    if constexpr (kPeer) {
        if (km == 8 && dyn)
            return f8 ? reduce_tcgen05_kernel<true, 8, true, true> : reduce_tcgen05_kernel<false, 8, true, true>;
        if (km == 8) return f8 ? reduce_tcgen05_kernel<true, 8, true> : reduce_tcgen05_kernel<false, 8, true>;
        return f8 ? reduce_tcgen05_kernel<true, 0, true> : reduce_tcgen05_kernel<false, 0, true>;
    } else {
        if (dyn) {
            switch (km) {
                case 4: return f8 ? reduce_tcgen05_kernel<true, 4, false, true> : reduce_tcgen05_kernel<false, 4, false, true>;
                case 8: return f8 ? reduce_tcgen05_kernel<true, 8, false, true> : reduce_tcgen05_kernel<false, 8, false, true>;
                case 16: if (!f8) return reduce_tcgen05_kernel<false, 16, false, true>; break;
                default: break;
            }
        }
        switch (km) {
            case 4: return f8 ? reduce_tcgen05_kernel<true, 4> : reduce_tcgen05_kernel<false, 4>;
            case 8: return f8 ? reduce_tcgen05_kernel<true, 8> : reduce_tcgen05_kernel<false, 8>;
            case 16: return f8 ? reduce_tcgen05_kernel<true, 16> : reduce_tcgen05_kernel<false, 16>;
            default: return f8 ? reduce_tcgen05_kernel<true, 0> : reduce_tcgen05_kernel<false, 0>;
        }
    }
}

// exact: the exact E4M3 entry -- the default ring (4 x 32 KiB, 4
// accumulators x chain 2: rows of 64 values, exact in binary32) and the
// integer combine (the dynamic-tail instantiation, with or without a tail);
// out_acc (may be null) receives the exact state.
template <bool kPeer>
static cudaError_t launch_tc05(int fmt, const uint8_t* x, size_t n, float* out_f32, double* out_f64,
                               const DevWorkspace& ws, const LaunchCfg& cfg_in, const PeerCombine& pc,
                               bool emulate, cudaStream_t stream, bool exact = false,
                               long long* out_acc = nullptr) {
    const size_t es = fmt >= 2 ? 1u : 2u;
    const int P = emulate ? pc.nranks : 1;
    LaunchCfg cfg0 = cfg_in;
    if (exact) {
        cfg0.tc05_stages = 4;
        cfg0.tc05_stage_kb = 32;
        cfg0.tc05_slots = 4;
        cfg0.tc05_chain = 2;
        cfg0.tc05_ctas = 0;
        cfg0.tc05_prefetch = 0;
        cfg0.tc05_split = 1;
        cfg0.tc05_interleave = 0;
    }
    const LaunchCfg cfg = tc05_effective(n / (size_t)P * es, cfg0);  // by the per-rank bytes
    Tc05Params prm;
    prm.fmt = fmt;
    prm.out_acc = out_acc;  // (exact only)
    // kind::f16: a/b_format F16 = 0, BF16 = 1; kind::f8f6f4: E4M3 = 0, E5M2 = 1 (bits 7-9, 10-12)
    const uint32_t ab = (fmt == 1 || fmt == 3) ? ((1u << 7) | (1u << 10)) : 0u;
    prm.idesc = kIdesc | ab;
    prm.one_bits = fmt == 1 ? 0x3F803F80u : fmt == 2 ? 0x38383838u : fmt == 3 ? 0x3C3C3C3Cu
                                                                   : 0x3C003C00u;
    prm.stages = cfg.tc05_stages;
    prm.stage_bytes = (uint32_t)cfg.tc05_stage_kb * 1024u;
    prm.slots = cfg.tc05_slots;
    prm.chain = cfg.tc05_chain;
    prm.prefetch = cfg.tc05_prefetch;
    prm.split = cfg.tc05_split;
    prm.interleave = cfg.tc05_interleave;
    prm.dynamic = cfg.tc05_dynamic;  // gated on the run length below
    if (prm.slots < 1 || prm.slots > 16 || (prm.slots & (prm.slots - 1)) || prm.chain < 1 ||
        prm.stage_bytes % kTileBytes || prm.stage_bytes % (16u * (uint32_t)prm.split))
        return cudaErrorInvalidValue;
    const size_t smem = kHeaderBytes + (size_t)prm.stages * prm.stage_bytes;
    if (kHeaderBytes - 8 < 512 + (size_t)(2 * prm.stages + 4) * 8 + (size_t)(prm.stages + 2) * 4)
        return cudaErrorInvalidValue;
    // one accumulator round per stage (4 slots, chain = MMAs per stage / 4):
    // the tight issue loop, instantiated for 4, 8 and 16 MMAs per stage
    const int kmma = (int)(prm.stage_bytes / kTileBytes);
    const int km = (prm.slots == 4 && prm.slots * prm.chain == kmma &&
                    (kmma == 4 || kmma == 8 || kmma == 16)) ? kmma : 0;
    // the dynamic tail: binary16 / fp8 (bfloat16 sums are not multiples of
    // 2^-24), the tight loop, fp8 up to 8 MMAs per stage, dynamic > 0, and
    // runs of at least cfg.tc05_dyn_min_run chunks per CTA (default 32:
    // shorter inputs lose more to the ticket latency than the tail costs,
    // 2^24 6.4 -> 9.4 us, profiles/r02/tc05_dyn_ab1.txt)
    const size_t chunks = n / (size_t)P * es / prm.stage_bytes;
    const bool dyn = prm.dynamic > 0 && fmt != 1 && km > 0 && (fmt < 2 || km <= 8) &&
                     (!kPeer || km == 8) &&
                     chunks >= (size_t)cfg.tc05_dyn_min_run * (size_t)tcgen05_grid(n / (size_t)P * es, cfg);
    if (!dyn) prm.dynamic = 0;
    if (exact && (fmt != 2 || (km != 8 && km != 4) || kPeer)) return cudaErrorInvalidValue;  // chain <= 2
    const bool dyn_inst = dyn || exact;  // exact: the integer combine even without a tail
    const Tc05Kernel kernel = tc05_kernel<kPeer>(fmt >= 2, km, dyn_inst);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        // largest dynamic shared memory size configured so far, per (device, kernel)
        static std::mutex mu;
        static std::map<std::pair<int, const void*>, size_t> configured;
        std::lock_guard<std::mutex> lk(mu);
        size_t& have = configured[{dev, (const void*)kernel}];
        if (smem > have) {
            if ((e = cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem)))
                return e;
            have = smem;
        }
    }
    int g = tcgen05_grid(n / (size_t)P * es, cfg);
    const dim3 block(kTcWarps * 32);
    if (!emulate) {
        // the peer variant waits on other ranks: plain launch
        launch_maybe_pdl(kernel, dim3(g), block, smem, stream, (cfg.pdl && !kPeer) ? 1 : 0, x, n, prm,
                         out_f32, out_f64, ws, pc);
        return cudaGetLastError();
    }
    // emulated peer group: the ranks' last CTAs wait on one another, so all P
    // grid slices must be co-resident -- a cooperative launch guarantees it
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kTcWarps * 32, smem)))
        return e;
    const int cap = occ * cfg.sms / P;
    if (g > cap) g = cap;
    if (g < 1) return cudaErrorCooperativeLaunchTooLarge;
    const uint8_t* xa = x;
    size_t na = n;
    Tc05Params pa = prm;
    float* o32 = out_f32;
    double* o64 = out_f64;
    DevWorkspace wsa = ws;
    PeerCombine pca = pc;
    void* args[] = {(void*)&xa, (void*)&na, (void*)&pa, (void*)&o32, (void*)&o64, (void*)&wsa,
                    (void*)&pca};
    return cudaLaunchCooperativeKernel((const void*)kernel, dim3(g, P), block, args, smem, stream);
}

cudaError_t launch_reduce_tcgen05(int fmt, const uint16_t* x16, size_t n, float* out_f32,
                                  double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                  cudaStream_t stream) {
    const PeerCombine none{};
    return launch_tc05<false>(fmt, reinterpret_cast<const uint8_t*>(x16), n, out_f32, out_f64, ws, cfg,
                              none, false, stream);
}

cudaError_t launch_reduce_tcgen05_peer(int fmt, const uint16_t* x16, size_t n, float* out_f32,
                                       double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                       const PeerCombine& pc, bool emulate, cudaStream_t stream) {
    return launch_tc05<true>(fmt, reinterpret_cast<const uint8_t*>(x16), n, out_f32, out_f64, ws, cfg,
                             pc, emulate, stream);
}

// NaN count for the exact E4M3 entry (runs after the reduction on the same
// stream): nothing to do unless the reduction marked acc[4] = -1 (a level-2
// total was NaN); then every CTA counts its share of the NaN bytes (0x7F /
// 0xFF) into acc[3] and the last CTA (ticket) clears the marker.
__global__ void e4m3_nan_count_kernel(const uint8_t* __restrict__ x, size_t n, long long* acc,
                                      DevWorkspace ws) {
    if (__ldcg(acc + 4) != -1) return;
    unsigned long long c = 0;
    const size_t T = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T)
        c += ((__ldg(x + i) & 0x7Fu) == 0x7Fu) ? 1u : 0u;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned s_last;
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(acc + 3), c);
    __syncthreads();
    if (threadIdx.x == 0) s_last = (ticket_acq_rel(ws.ticket) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        acc[4] = 0;
        *ws.ticket = 0u;
    }
}

bool exact_e4m3_tc05_applies(size_t n, const LaunchCfg& cfg) {
    return cfg.exact_bulk != 0 && n >= ((size_t)64 << 20);
}

cudaError_t launch_exact_e4m3_tc05(const uint8_t* x, size_t n, long long* out_acc, float* out_f32,
                                   double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                   cudaStream_t stream, int* launches) {
    const PeerCombine none{};
    cudaError_t e = launch_tc05<false>(2, x, n, out_f32, out_f64, ws, cfg, none, false, stream, true, out_acc);
    *launches = 1;
    if (e != cudaSuccess || !out_acc) return e;
    e4m3_nan_count_kernel<<<cfg.sms * 2, 256, 0, stream>>>(x, n, out_acc, ws);
    *launches = 2;
    return cudaGetLastError();
}

// One tcgen05.mma (M=128, N=16, K=16) with A = a (row-major 128x16 fp16),
// B = ones, C[r][*] = c[r] written into TMEM with tcgen05.st; d[r] = D[r][0].
// Element (r, k) of A is placed at byte (r/8)*256 + (k/8)*128 + (r%8)*16 +
// (k%8)*2 -- the layout the reduction's descriptor (LBO=128, SBO=256) names.
__global__ void __launch_bounds__(128) probe_tcgen05_kernel(const uint16_t* a, const float* c,
                                                            float* d) {
    __shared__ __align__(1024) uint16_t sa[128 * 16];
    __shared__ __align__(1024) uint16_t sb[256];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 16; i += 128) {
        const int r = i / 16, k = i % 16;
        sa[((r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) / 2] = a[i];
    }
    for (int i = tid; i < 256; i += 128) sb[i] = 0x3C00;
    sm100::fence_proxy_async_smem();
    if (tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
    }
    if (warp == 0) sm100::tmem_alloc(&tbase, 32);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t cv[16];
    for (int j = 0; j < 16; ++j) cv[j] = __float_as_uint(c[tid]);
    sm100::tmem_st_32x32b_x16(lane_addr, cv);
    sm100::tmem_wait_st();
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    if (tid == 0) {
        sm100::mma_f16_ss(tmem, sm100::smem_desc_kmajor(sm100::smem_addr(sa), 128, 256),
                          sm100::smem_desc_kmajor(sm100::smem_addr(sb), 128, 256), kIdesc, 1u);
        sm100::mma_commit(&bar);
    }
    sm100::mbar_wait(&bar, 0);
    sm100::tc_fence_after();
    const uint32_t r = sm100::tmem_ld_32x32b_x1(lane_addr);
    sm100::tmem_wait_ld();
    d[tid] = __uint_as_float(r);
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) sm100::tmem_dealloc(tmem, 32);
}

cudaError_t launch_probe_mma_tcgen05(const uint16_t* a, const float* c, float* d,
                                     cudaStream_t stream) {
    probe_tcgen05_kernel<<<1, 128, 0, stream>>>(a, c, d);
    return cudaGetLastError();
}

}  // namespace tcr
