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

#ifndef TCR_SEG_BATCH
#define TCR_SEG_BATCH 8
#endif
#ifndef TCR_SEG_UNROLL
#define TCR_SEG_UNROLL 8
#endif
#ifndef TCR_SEG_CTAS
#define TCR_SEG_CTAS 4
#endif
constexpr unsigned long long kBatchSeg = TCR_SEG_BATCH;  // segments per scheduler atomic (guided)

// Reduce elements [s, e) of the 16-byte-aligned array xb (element indices
// relative to xb).  Returns the lane's fp64 share; the sum over lanes is the
// segment total.
// A warp takes a batch of consecutive segments (one global atomic per batch,
// guided self-scheduling) and streams the CONTIGUOUS union of the batch in
// groups of U tiles (one memory round trip each, all loads issued before the
// first MMA).  Each 256-element tile is attributed to the segments it
// overlaps, in order: a tile inside the current segment is one MMA
// (D = A x 1, C = 0 -- the paper's per-group formulation); a tile
// crossing a boundary gets one zero-masked MMA per overlapped segment (the
// paper's zero padding, reading G5); when a segment ends its row sums are
// collapsed (D' = 1 x D, three DMMAs) and written to out[j].  Long segments
// therefore stream at full width and many short segments share a round trip.
// The next batch's index and offsets are fetched during the current batch.
// F = element format (binary16, bfloat16, fp8 E4M3 / E5M2): a 16-byte vector
// holds EPV = 16 / bytes elements and a 512-byte tile 32 * EPV; all element
// indices below are in elements of that format.
template <bool kMma, int F>
__device__ __forceinline__ void seg_piece(const uint4& v, double& acc, int lane) {
    if constexpr (kMma) {
        float c[4] = {0.f, 0.f, 0.f, 0.f};
        mma_rowsum_f<F>(c, v);
        flush_rows(c, acc, lane);
    } else {
        acc += (double)vec_sum_f<F>(v);
    }
}

// Resident CTAs per SM of the union-stream kernel (__launch_bounds__): 4 for
// CSR (64 registers); 3 for fixed-length batches, whose 64-bit segment
// arithmetic needs the room (85 registers: zero spills, ptxas report).
template <bool kBatched>
constexpr int seg_resident() { return kBatched ? 3 : TCR_SEG_CTAS; }

template <bool kMma, int F, bool kBatched, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, seg_resident<kBatched>())
reduce_segmented_kernel(const uint8_t* __restrict__ x, const int64_t* __restrict__ offsets,
                        size_t S, size_t L, int batch, float* __restrict__ out, DevWorkspace ws) {
    pdl_wait_and_release();
    constexpr int kLogEpv = FmtInfo<F>::kBytes == 2 ? 3 : 4;  // log2(elements per vector)
    constexpr int64_t kEpv = (int64_t)1 << kLogEpv;
    constexpr int64_t kTileEl = 32 * kEpv;                     // elements per 512-byte tile
    const int lane = threadIdx.x & 31;
    const uintptr_t addr = (uintptr_t)x;
    const int64_t shift = (int64_t)((addr & 15u) / FmtInfo<F>::kBytes);
    const uint4* xb = reinterpret_cast<const uint4*>(addr & ~(uintptr_t)15u);
    const unsigned total_warps = gridDim.x * WARPS;
    const unsigned long long tail_zone = 2ull * total_warps * (unsigned long long)batch;
    const unsigned long long kIdx = (1ull << 56) - 1;

    auto grab = [&](unsigned long long hint) -> unsigned long long {  // lane 0 holds the result
        unsigned long long got = 0;
        const unsigned long long b = (S > hint + tail_zone) ? (unsigned long long)batch : 1ull;
        if (lane == 0) got = atomicAdd(ws.seg_next, b) | (b << 56);
        return got;
    };
    // CSR: lane k <= nb holds offsets[jb + k] + shift (one load per lane per batch)
    auto load_offs = [&](unsigned long long jb, int nb) -> int64_t {
        if constexpr (kBatched) {
            return 0;
        } else {
            return (lane <= nb && jb + lane <= S) ? __ldg(offsets + jb + lane) + shift : 0;
        }
    };
    unsigned long long g = __shfl_sync(0xffffffffu, grab(0), 0);
    unsigned long long jb = g & kIdx;
    int nb = (int)(g >> 56);
    unsigned long long pend = grab(jb);
    int64_t offl = load_offs(jb, nb);

    while (jb < S) {
        if ((unsigned long long)nb > S - jb) nb = (int)(S - jb);
        auto off = [&](int k) -> int64_t {  // start of segment jb + k (k <= nb), element units
            if constexpr (kBatched) return (int64_t)((jb + (unsigned long long)k) * L) + shift;
            else return __shfl_sync(0xffffffffu, offl, k);
        };
        // the next batch: index now, offsets in flight during this batch
        const unsigned long long p = __shfl_sync(0xffffffffu, pend, 0);
        const unsigned long long jb2 = p & kIdx;
        const int nb2 = (int)(p >> 56);
        pend = grab(jb2);
        const int64_t offl2 = (jb2 < S) ? load_offs(jb2, nb2) : 0;

        const int64_t r0 = off(0), r1 = off(nb);
        // Tiles sit on absolute 256-element boundaries (relative to xb), so the
        // arithmetic of a segment never depends on which batch / warp reduced
        // it (bitwise determinism under dynamic scheduling).
        const int64_t Vlo = r0 >> kLogEpv, V1 = (r1 + kEpv - 1) >> kLogEpv;
        const int64_t V0 = Vlo & ~(int64_t)31;
        int cs = 0;
        int64_t sb = r0, se = off(1);
        double acc = 0.0;
        for (int64_t vb = V0; vb < V1; vb += 32 * U) {
            uint4 v[U];
            const int64_t f0 = (r0 + kEpv - 1) >> kLogEpv, f1 = r1 >> kLogEpv;
            if (vb >= f0 && vb + 32 * U <= f1) {
#pragma unroll
                for (int u = 0; u < U; ++u) v[u] = ldg_stream(xb + vb + u * 32 + lane);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t vi = vb + u * 32 + lane;
                    v[u] = make_uint4(0u, 0u, 0u, 0u);
                    if (vi >= Vlo && vi < V1)
                        v[u] = mask_vec_f<F>(ldg_stream(xb + vi), vi * kEpv, r0, r1);
                }
            }
            __syncwarp();  // scheduling fence: all U loads issue before the first consumer
            const int64_t g0 = vb * kEpv, g1 = g0 + (int64_t)U * kTileEl;
            if (cs < nb && sb <= g0 && se > g1) {
                // the whole group lies inside segment cs (the common case for long
                // segments): U independent tiles, no per-tile control flow; each
                // tile is its own MMA with C = 0, flushed in tile order
                if constexpr (kMma) {
                    float c[U][4];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        c[u][0] = c[u][1] = c[u][2] = c[u][3] = 0.f;
                        mma_rowsum_f<F>(c[u], v[u]);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) flush_rows(c[u], acc, lane);
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) acc += (double)vec_sum_f<F>(v[u]);
                }
                continue;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t t0 = (vb + u * 32) * kEpv, t1 = t0 + kTileEl;  // tile elements
                if (t0 >= r1) break;
                while (cs < nb) {
                    if (sb >= t1) break;  // current segment starts after this tile
                    if (sb <= t0 && se >= t1) {  // tile entirely inside segment cs
                        seg_piece<kMma, F>(v[u], acc, lane);
                    } else if (se > sb && se > t0) {  // the part of the tile inside [sb, se)
                        seg_piece<kMma, F>(mask_vec_f<F>(v[u], (vb + u * 32 + lane) * kEpv, sb, se),
                                           acc, lane);
                    }
                    if (se > t1) break;  // segment continues in the next tile
                    const double tot = warp_collapse<kMma>(acc);  // segment cs ends in this tile
                    if (lane == 0) out[jb + cs] = (float)tot;
                    acc = 0.0;
                    ++cs;
                    sb = se;
                    if (cs < nb) se = off(cs + 1);
                }
            }
        }
        for (; cs < nb; ++cs) {  // trailing (empty) segments of the batch
            const double tot = warp_collapse<kMma>(acc);
            if (lane == 0) out[jb + cs] = (float)tot;
            acc = 0.0;
        }
        jb = jb2;
        nb = nb2;
        offl = offl2;
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

// Fixed-length rows of T whole 512-byte tiles (L = T * tile elements, T in
// {1, 2, 4, 8}, x 16-byte aligned): every group of 8 tiles holds 8/T complete rows, so a warp issues
// its 8 loads, 8 independent MMAs (C = 0), folds them per row and collapses
// the 8/T rows with no data-dependent control flow.  Rows are dealt to warps
// statically (all rows cost the same: no scheduler, no atomics).
template <bool kMma, int F, int T, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4)
reduce_rows_kernel(const uint8_t* __restrict__ x, size_t S, float* __restrict__ out) {
    pdl_wait_and_release();
    constexpr int R = 8 / T;  // rows per group
    const int lane = threadIdx.x & 31;
    const uint4* xv = reinterpret_cast<const uint4*>(x) + lane;
    const size_t groups = (S + R - 1) / R;
    const size_t W = (size_t)gridDim.x * WARPS;
    for (size_t gi = (size_t)blockIdx.x * WARPS + (threadIdx.x >> 5); gi < groups; gi += W) {
        const size_t row0 = gi * R;
        const int rows = (int)((S - row0) < (size_t)R ? (S - row0) : (size_t)R);
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            v[u] = make_uint4(0u, 0u, 0u, 0u);
            if (u / T < rows) v[u] = ldg_stream(xv + (row0 * T + u) * 32);
        }
        __syncwarp();  // scheduling fence: all loads issue before the first consumer
        double acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if constexpr (kMma) {
                float c[4] = {0.f, 0.f, 0.f, 0.f};
                mma_rowsum_f<F>(c, v[u]);
                flush_rows(c, acc[u / T], lane);
            } else {
                acc[u / T] += (double)vec_sum_f<F>(v[u]);
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double tot = warp_collapse<kMma>(acc[r]);
            if (lane == 0 && r < rows) out[row0 + r] = (float)tot;
        }
    }
}

// Fixed-length rows as MMA rows (r02): 16 consecutive segments fill the 16
// rows of A, so the row sums of Eq. 9-10 (D = A x 1 + C) ARE per-segment
// partial sums -- no second-level collapse per segment.  In the paper one
// group of m^2 inputs fills A and D' = 1 x D collapses its rows;
// here the rows belong to different segments and stay apart.  Each row takes
// 16 elements of its segment per MMA; C is carried over the segment's MMAs
// (bounded chain: flushed into fp64 every kRsChain MMAs, reading G9).
// Fragment use (m16n8k16, lane 4g + t): a0 = A[g][2t..], a1 = A[g+8][2t..],
// a2 = A[g][2t+8..], a3 = A[g+8][2t+8..].  Lane 4g + t loads 16 bytes
// (8 values) of segment g and 16 of segment g + 8 at element 32p + 8t: values
// 0-3 feed MMA 2p, 4-7 MMA 2p + 1, so every row of A gets 16 elements of its
// own segment (a bijection of the segment's elements onto its A rows, reading
// G1).  Lanes 4g..4g+3 read 64 contiguous bytes per segment per load round.
// D: c0 = c1 = row g, c2 = c3 = row g + 8 in every lane of quad g.  Needs
// L % 32 == 0 (whole MMA pairs) and a 16-byte aligned x; 16-bit formats.
constexpr int kRsChain = 4;  // MMAs per fp32 chain before the fp64 flush (K = 4, reading G10)

// P = MMA pairs in flight per lane (2 loads each): 4 from L = 128 (the whole
// row span up to 2048 in rounds of 256 B per row), else the row's own pair
// count -- no dead load slots for short rows (measured, scripts/ab_rows.py:
// L = 64 at P = 4: 5.9 TB/s, at P = 2: 6.7 TB/s).
constexpr int kRsCtasPerSm = 3;  // resident CTAs per SM (<= 85 registers: no spills at P <= 4)

template <int F, int WARPS, int P>
__global__ void __launch_bounds__(WARPS * 32, kRsCtasPerSm)
reduce_rowseg_kernel(const uint8_t* __restrict__ x, size_t S, size_t L, float* __restrict__ out) {
    pdl_wait_and_release();
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const size_t slabs = (S + 15) / 16;
    const size_t W = (size_t)gridDim.x * WARPS;
    const size_t pairs = L / 32;  // 32 elements (64 bytes) of a row per MMA pair
    for (size_t sl = (size_t)blockIdx.x * WARPS + (threadIdx.x >> 5); sl < slabs; sl += W) {
        const size_t r0 = sl * 16 + (size_t)g, r1 = r0 + 8;
        const bool in0 = r0 < S, in1 = r1 < S;
        const uint4* p0 = reinterpret_cast<const uint4*>(x + r0 * L * 2) + t;  // row r1 = p0 + L
        double acc0 = 0.0, acc1 = 0.0;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (size_t p = 0; p < pairs; p += P) {
            uint4 lo[P], hi[P];
#pragma unroll
            for (int u = 0; u < P; ++u) {
                const bool in = p + (size_t)u < pairs;
                lo[u] = (in && in0) ? ldg_stream(p0 + (p + (size_t)u) * 4) : make_uint4(0u, 0u, 0u, 0u);
                hi[u] = (in && in1) ? ldg_stream(p0 + L + (p + (size_t)u) * 4) : make_uint4(0u, 0u, 0u, 0u);
            }
            __syncwarp();  // scheduling fence: all loads issue before the first MMA
#pragma unroll
            for (int u = 0; u < P; ++u) {
                mma_rowsum_f<F>(c, make_uint4(lo[u].x, hi[u].x, lo[u].y, hi[u].y));
                mma_rowsum_f<F>(c, make_uint4(lo[u].z, hi[u].z, lo[u].w, hi[u].w));
                if ((2 * u + 2) % kRsChain == 0 || u == P - 1) {  // <= kRsChain MMAs per chain (static)
                    // every lane of quad g holds rows g / g + 8 (no branch)
                    acc0 += (double)c[0];
                    acc1 += (double)c[2];
                    c[0] = c[1] = c[2] = c[3] = 0.f;
                }
            }
        }
        acc0 += (double)c[0];
        acc1 += (double)c[2];
        if (t == 0) {
            if (in0) out[r0] = (float)acc0;
            if (in1) out[r1] = (float)acc1;
        }
    }
}

constexpr int kSegWarps = 8;
constexpr int kSegUnroll = TCR_SEG_UNROLL;  // tiles per group (one round trip)
constexpr int kSegCtasPerSm = TCR_SEG_CTAS;  // resident CTAs per SM (launch bounds: 64 registers at 4)

template <bool kMma, int F>
static void launch_seg_t(bool batched, const dim3& grid, const dim3& block, const uint8_t* x,
                         const int64_t* offsets, size_t S, size_t L, float* out,
                         const DevWorkspace& ws, cudaStream_t stream, int sms, int pdl) {
    constexpr size_t kTileEl = 512 / FmtInfo<F>::kBytes;
    if constexpr (kMma && FmtInfo<F>::kBytes == 2) {
        // fixed-length rows of 32..2048 binary16 / bfloat16: rows as MMA rows,
        // except L = 1024 / 2048, where the whole-tile rows kernel below
        // measured faster (6.9 vs 6.5 TB/s; profiles/r02/batched_b2b.txt)
        if (batched && ((uintptr_t)x & 15u) == 0 && L % 32 == 0 && L >= 32 && L <= 2048 &&
            L != 4 * kTileEl && L != 8 * kTileEl) {
            const size_t slabs = (S + 15) / 16;
            const size_t pairs = L / 32;
            size_t g = (slabs + kSegWarps - 1) / kSegWarps;
            // P <= 2 needs <= 46 registers: 5 CTAs per SM fit (more loads in flight)
            const size_t gmax = (size_t)sms * (pairs >= 4 ? kRsCtasPerSm : 5);
            if (g > gmax) g = gmax;
            if (g < 1) g = 1;
            const dim3 rg((unsigned)g);
            if (pairs >= 4)
                launch_maybe_pdl(reduce_rowseg_kernel<F, kSegWarps, 4>, rg, block, 0, stream, pdl, x, S, L, out);
            else if (pairs >= 2)
                launch_maybe_pdl(reduce_rowseg_kernel<F, kSegWarps, 2>, rg, block, 0, stream, pdl, x, S, L, out);
            else
                launch_maybe_pdl(reduce_rowseg_kernel<F, kSegWarps, 1>, rg, block, 0, stream, pdl, x, S, L, out);
            return;
        }
    }
    if (batched && ((uintptr_t)x & 15u) == 0 &&
        (L == kTileEl || L == 2 * kTileEl || L == 4 * kTileEl || L == 8 * kTileEl)) {
        const size_t rows_per_group = 8 * kTileEl / L;
        const size_t groups = (S + rows_per_group - 1) / rows_per_group;
        size_t g = (groups + kSegWarps - 1) / kSegWarps;
        const size_t gmax = (size_t)sms * kSegCtasPerSm;
        if (g > gmax) g = gmax;
        if (g < 1) g = 1;
        const dim3 rgrid((unsigned)g);
        switch (L / kTileEl) {
            case 1: launch_maybe_pdl(reduce_rows_kernel<kMma, F, 1, kSegWarps>, rgrid, block, 0, stream, pdl, x, S, out); break;
            case 2: launch_maybe_pdl(reduce_rows_kernel<kMma, F, 2, kSegWarps>, rgrid, block, 0, stream, pdl, x, S, out); break;
            case 4: launch_maybe_pdl(reduce_rows_kernel<kMma, F, 4, kSegWarps>, rgrid, block, 0, stream, pdl, x, S, out); break;
            default: launch_maybe_pdl(reduce_rows_kernel<kMma, F, 8, kSegWarps>, rgrid, block, 0, stream, pdl, x, S, out); break;
        }
        return;
    }
    if (batched) {
        // ~32 KiB per batch for short fixed lengths, at least 8 segments
        size_t b = L ? ((size_t)32768 / FmtInfo<F>::kBytes / L) : 255;
        if (b < kBatchSeg) b = kBatchSeg;
        if (b > 255) b = 255;
        dim3 bgrid = grid;  // one resident wave at this kernel's occupancy
        const unsigned bmax = (unsigned)(sms * seg_resident<true>());
        if (bgrid.x > bmax) bgrid.x = bmax;
        launch_maybe_pdl(reduce_segmented_kernel<kMma, F, true, kSegUnroll, kSegWarps>, bgrid, block, 0,
                         stream, pdl, x, offsets, S, L, (int)b, out, ws);
    } else {
        launch_maybe_pdl(reduce_segmented_kernel<kMma, F, false, kSegUnroll, kSegWarps>, grid, block, 0,
                         stream, pdl, x, offsets, S, L, (int)kBatchSeg, out, ws);
    }
}

template <bool kMma>
static void launch_seg_m(int fmt, bool batched, const dim3& grid, const dim3& block,
                         const uint8_t* x, const int64_t* offsets, size_t S, size_t L, float* out,
                         const DevWorkspace& ws, cudaStream_t stream, int sms, int pdl) {
    switch (fmt) {
        case kBF16: launch_seg_t<kMma, kBF16>(batched, grid, block, x, offsets, S, L, out, ws, stream, sms, pdl); break;
        case kE4M3: launch_seg_t<kMma, kE4M3>(batched, grid, block, x, offsets, S, L, out, ws, stream, sms, pdl); break;
        case kE5M2: launch_seg_t<kMma, kE5M2>(batched, grid, block, x, offsets, S, L, out, ws, stream, sms, pdl); break;
        default: launch_seg_t<kMma, kF16>(batched, grid, block, x, offsets, S, L, out, ws, stream, sms, pdl); break;
    }
}

cudaError_t launch_reduce_segmented(bool mma, int fmt, bool batched, const void* x,
                                    const int64_t* offsets, size_t num_segments,
                                    size_t segment_len, float* out, const DevWorkspace& ws,
                                    const LaunchCfg& cfg, cudaStream_t stream) {
    // fixed-length rows on tcgen05 (tcr_rows_tc05.cu) when every SM gets a
    // block of 256 segments and L <= 3072, except L = 1024, where the
    // whole-tile mma.sync rows kernel measured faster (1 GiB inputs,
    // profiles/r02/rows_tc05_sweep.txt, rows_tc05_sweep2.txt: tcgen05 0.89-
    // 0.98 x the mma.sync kernels' time for L = 32..768, 2048, 3072; 0.03-
    // 0.13 x for L = 8..56 other than 32, which had no specialised kernel;
    // 1.03 x at 1024, 1.04 x at 4096)
    const size_t L = segment_len;
    if (mma && batched && cfg.rows_tc05 && num_segments >= (size_t)256 * (size_t)cfg.sms &&
        L * ((fmt == kE4M3 || fmt == kE5M2) ? 1 : 2) <= 6144 && !(fmt <= kBF16 && L == 1024) &&
        rows_tc05_supported(fmt, x, num_segments, L))
        return launch_reduce_rows_tc05(fmt, x, num_segments, segment_len, out, ws, cfg, stream);
    size_t g = (num_segments + kSegWarps - 1) / kSegWarps;
    const size_t gmax = (size_t)cfg.sms * kSegCtasPerSm;
    if (g > gmax) g = gmax;
    if (g < 1) g = 1;
    const dim3 grid((unsigned)g), block(kSegWarps * 32);
    const uint8_t* xb = static_cast<const uint8_t*>(x);
    if (mma)
        launch_seg_m<true>(fmt, batched, grid, block, xb, offsets, num_segments, segment_len, out, ws,
                           stream, cfg.sms, cfg.pdl);
    else
        launch_seg_m<false>(fmt, batched, grid, block, xb, offsets, num_segments, segment_len, out, ws,
                            stream, cfg.sms, cfg.pdl);
    return cudaGetLastError();
}

}  // namespace tcr
