// tcr_rows_tc05.cu -- fixed-length segments (tcr_reduce_sum_batched) on the
// 5th-generation tensor cores, segments as the rows of A:
//
//   HBM --(TMA tensor copy: 2-D map {L, S}, box {BW elements, 256 rows},
//   32 / 64 / 128-byte swizzle for BW = 16 / 32 / 64)--> 32 KiB SMEM stage
//   (64 / BW boxes) in the canonical swizzled K-major UMMA layout --(8 x
//   tcgen05.mma M128 N16 K16 per stage: two 128-row halves per box, the K
//   slices at +32 B, B = ones)--> fp32 TMEM accumulators --(tcgen05.ld, one
//   row per thread per half)--> binary64 per segment --> out[j].
//
// Paper mapping (arXiv 1903.03640): D = A x 1 (Eq. 9-10) with row
// r of A holding BW elements of segment r: "the m row sums" are the segment
// partial sums directly, so no D' = 1 x D collapse per segment is needed --
// the collapse that recombines one group's row sums (Eq. 11-12) has nothing
// to do when every row is a different segment.  A box's K slices (<= 4
// MMAs) are the carried chain (K <= 4, reading G9); each box's row sums are
// flushed into binary64 (bounded truncation, reading G10).  A segment's
// boxes are added in index order by one thread: deterministic, independent
// of the grid.  The box width is the narrowest of 16 / 32 / 64 that holds
// a whole short segment (L <= 16 / 32), so short rows do not fetch and
// multiply 64-element boxes that are mostly zero fill.
//
// The tensor map's out-of-bounds fill supplies the paper's zero padding of
// the trailing group (reading G5): elements past L (L not a multiple of BW)
// and rows past S arrive as zeros.
//
// Warp roles (192 threads): warp 0 lane 0 producer (TMA), warp 1 lane 0 MMA
// issuer (warp 1 allocates TMEM), warps 2-5 epilogue (TMEM lane quarter
// warp % 4: rows 32 (warp % 4) .. + 31 of both halves of every box).
// 256-row boxes (8 MMAs per stage) rather than 128-row ones: the issuing
// thread's per-box bookkeeping (two barrier waits, a commit pair, the block
// hand-off) was the limit at 16 KiB per box.
#include <cuda.h>

#include <map>
#include <mutex>

#include "tcr_device.cuh"
#include "tcr_internal.h"
#include "tcr_sm100.cuh"

namespace tcr {

namespace {

constexpr int kRtWarps = 6;
constexpr int kRtRows = 256;                     // segments per box = 2 x M
constexpr uint32_t kRtStageBytes = 32768;        // one ring stage (64 / BW boxes)
constexpr uint32_t kRtHeader = 1024;             // ones tile + barriers + TMEM address
constexpr int kRtAcc = 4;                        // TMEM accumulator buffers

// Box geometry by box width BW (elements of a segment per box): 64 (L > 32,
// 128-byte rows, SWIZZLE_128B), 32 (L <= 32, SWIZZLE_64B) or 16 (L <= 16,
// SWIZZLE_32B).  A stage holds 64 / BW boxes of 256 rows; every box is two
// 128-row halves (two M = 128 MMAs per K slice of 16 elements), and every
// stage is 8 MMAs.  Boxes narrower than 64 cover a whole segment (L <= BW),
// so a stage then completes 64 / BW row blocks.
template <int BW>
struct RtGeom {
    static constexpr int kNB = 64 / BW;                           // boxes per stage
    static constexpr uint32_t kBoxBytes = (uint32_t)BW * 2u * kRtRows;
    static constexpr uint32_t kHalfBytes = kBoxBytes / 2u;        // 128 rows
    static constexpr int kSlices = BW / 16;                       // K slices per box half
    static constexpr uint32_t kRowBytes = (uint32_t)BW * 2u;      // swizzle width
    static constexpr uint64_t kLayout = BW == 64 ? 2 : BW == 32 ? 4 : 6;  // SW128 / SW64 / SW32
    static constexpr uint32_t kCols = (uint32_t)kRtAcc * (uint32_t)kNB * 32u;  // TMEM columns
};

// K-major, swizzled UMMA descriptor of a 128-row SMEM tile written by a TMA
// box with the matching swizzle: 8-row atoms of 8 x kRowBytes (SBO), rows of
// kRowBytes inside an atom, the XOR swizzle applied by the hardware on
// address bits; LBO unused (1); version 1 (sm_100); layout type 2 / 4 / 6 =
// SWIZZLE_128B / 64B / 32B.  The K slice k (16 elements = 32 B) starts 32 k
// bytes into the tile.
template <int BW>
__device__ __forceinline__ uint64_t smem_desc_sw(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;                                    // LBO (ignored for swizzled K-major)
    d |= (uint64_t)((8u * RtGeom<BW>::kRowBytes) >> 4) << 32;  // SBO: 8 rows
    d |= (uint64_t)1 << 46;                                    // descriptor version (sm_100)
    d |= RtGeom<BW>::kLayout << 61;
    return d;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(sm100::smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sm100::smem_addr(bar))
        : "memory");
}

struct RtParams {
    size_t S;        // segments
    int nk;          // stages per unit = ceil(L / BW) (1 when BW < 64)
    int stages;      // SMEM ring stages
    uint32_t idesc;  // kind::f16 instruction descriptor (F16 or BF16 operands)
    uint32_t one_bits;
    long long dyn;   // units handed out by ticket at the end (the dynamic tail)
};

// A unit is 64 / BW consecutive row blocks of 256 segments (one stage per K
// box of them).  Units [0, Us) are dealt in grid-stride order, the last
// `dyn` units one at a time from ws.chunk_next (two tickets held ahead), as
// the flat kernel's dynamic tail (§16): every segment is reduced by one CTA
// in box order, so the schedule cannot change a bit.  The producer writes
// each stage's unit index (-1 = END) next to the stage; the MMA issuer
// forwards it per accumulator buffer with a plain arrive on tinf[a]
// (release), which the epilogue waits on before reading it.
// kF8: fp8 E4M3 / E5M2 rows (kind::f8f6f4, K = 32 one-byte elements per
// slice): the same byte geometry, BW counting 2-byte units.
template <int BW, bool kF8>
__global__ void __launch_bounds__(kRtWarps * 32)
reduce_rows_tc05_kernel(const __grid_constant__ CUtensorMap map, RtParams prm, float* __restrict__ out,
                        DevWorkspace ws) {
    using Geo = RtGeom<BW>;
    constexpr int kNB = Geo::kNB;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int stages = prm.stages;
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem);        // 512 B of ones (B operand)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 512);  // [stages]
    uint64_t* empty = full + stages;                           // [stages]
    uint64_t* tfull = empty + stages;                          // [kRtAcc]
    uint64_t* tempty = tfull + kRtAcc;                         // [kRtAcc]
    uint64_t* tinf = tempty + kRtAcc;                          // [kRtAcc]
    volatile int* sinfo = reinterpret_cast<volatile int*>(tinf + kRtAcc);  // [stages]
    volatile int* tinfo = sinfo + stages;                                  // [kRtAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kRtHeader - 8);
    uint8_t* ring = smem + kRtHeader;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const long long units = (long long)((prm.S + (size_t)kRtRows * kNB - 1) / ((size_t)kRtRows * kNB));
    const long long Us = units - prm.dyn;
    const long long G = gridDim.x, b = blockIdx.x;
    // static part in grid-stride order (CTA b: units b, b + G, ... < Us): at
    // any moment the grid reads neighbouring units (contiguous runs per CTA
    // measured ~10 % slower, profiles/r02/rows_tc05_ab2.txt)
    const long long n_static = b < Us ? (Us - b + G - 1) / G : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < kRtAcc; ++a) {
            sm100::mbar_init(&tfull[a], 1);
            sm100::mbar_init(&tempty[a], 4);
            sm100::mbar_init(&tinf[a], 1);
        }
        sm100::fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    }
    for (int i = threadIdx.x; i < 128; i += blockDim.x) ones[i] = prm.one_bits;
    sm100::fence_proxy_async_smem();
    constexpr uint32_t kCols = Geo::kCols;
    constexpr uint32_t kBufCols = kCols / kRtAcc;  // one stage's 2 kNB accumulators
    if (warp == 1) sm100::tmem_alloc(tmem_slot, kCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait_and_release();  // the previous kernel's writes (x, out, counters) visible

    if (warp == 0) {
        if (lane == 0) {  // producer: nk stages of kNB TMA boxes per unit, then END
            int s = 0;
            uint32_t ph = 0;
            auto unit_stages = [&](long long u) {
                for (int k = 0; k < prm.nk; ++k) {
                    sm100::mbar_wait(&empty[s], ph ^ 1u);
                    sinfo[s] = (int)u;
                    sm100::mbar_arrive_expect_tx(&full[s], kRtStageBytes);
                    for (int bx = 0; bx < kNB; ++bx)
                        tma_load_2d(ring + (size_t)s * kRtStageBytes + (size_t)bx * Geo::kBoxBytes, &map,
                                    k * BW * (kF8 ? 2 : 1), (int)((u * kNB + bx) * kRtRows), &full[s]);
                    if (++s == stages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
            };
            unsigned t0 = 0u, t1 = 0u;
            bool f0 = false, f1 = false;
            for (long long i = 0; i < n_static; ++i) {
                if (prm.dyn && !f0 && n_static - i <= 2) {
                    t0 = atomicAdd(ws.chunk_next, 1u);
                    f0 = true;
                }
                if (prm.dyn && !f1 && n_static - i <= 1) {
                    t1 = atomicAdd(ws.chunk_next, 1u);
                    f1 = true;
                }
                unit_stages(b + i * G);
            }
            if (prm.dyn) {
                if (!f0) t0 = atomicAdd(ws.chunk_next, 1u);
                if (!f1) t1 = atomicAdd(ws.chunk_next, 1u);
                for (;;) {
                    const unsigned t = t0;
                    t0 = t1;
                    t1 = atomicAdd(ws.chunk_next, 1u);
                    if ((long long)t >= prm.dyn) break;
                    unit_stages(Us + (long long)t);
                }
            }
            sm100::mbar_wait(&empty[s], ph ^ 1u);  // END: a stage with no bytes
            sinfo[s] = -1;
            sm100::mbar_arrive(&full[s]);
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer: 8 MMAs per stage into accumulator buffer j % kRtAcc
            const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
            const uint64_t adesc0 = smem_desc_sw<BW>(sm100::smem_addr(ring));
            constexpr uint64_t kStageStep = kRtStageBytes >> 4;
            int s = 0;
            uint32_t ph = 0;
            for (long long j = 0;; ++j) {
                const int a = (int)(j % kRtAcc);
                const uint32_t use = (uint32_t)(j / kRtAcc);
                sm100::mbar_wait(&full[s], ph);
                const int u = sinfo[s];
                sm100::mbar_wait(&tempty[a], (use & 1u) ^ 1u);  // drained kRtAcc stages ago
                tinfo[a] = u;
                if (u < 0) {
                    sm100::mbar_arrive(&tinf[a]);
                    break;
                }
                sm100::tc_fence_after();
                const uint64_t ad = adesc0 + (uint64_t)s * kStageStep;
                const uint32_t d = tmem + (uint32_t)a * kBufCols;
#pragma unroll
                for (int bx = 0; bx < kNB; ++bx)
#pragma unroll
                    for (int h = 0; h < 2; ++h)  // rows 128 h .. 128 h + 127 of the box
#pragma unroll
                        for (int q = 0; q < Geo::kSlices; ++q) {  // K slice q: +32 B = +2 in the descriptor
                            const uint64_t aq = ad + (uint64_t)((bx * Geo::kBoxBytes + h * Geo::kHalfBytes) >> 4) +
                                                (uint64_t)(2 * q);
                            if constexpr (kF8)
                                sm100::mma_f8_ss(d + 16u * (uint32_t)(2 * bx + h), aq, bdesc, prm.idesc, q > 0 ? 1u : 0u);
                            else
                                sm100::mma_f16_ss(d + 16u * (uint32_t)(2 * bx + h), aq, bdesc, prm.idesc, q > 0 ? 1u : 0u);
                        }
                sm100::mma_commit(&tfull[a]);
                sm100::mma_commit(&empty[s]);
                sm100::mbar_arrive(&tinf[a]);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        __syncwarp();
    } else {  // epilogue: rows r = 32 (warp % 4) + lane and r + 128 of every box
        const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
        const int row = (int)quarter + lane;
        double acc[2 * kNB];
#pragma unroll
        for (int i = 0; i < 2 * kNB; ++i) acc[i] = 0.0;
        int k = 0;
        for (long long j = 0;; ++j) {
            const int a = (int)(j % kRtAcc);
            const uint32_t use = (uint32_t)(j / kRtAcc);
            sm100::mbar_wait(&tinf[a], use & 1u);
            const int u = tinfo[a];
            if (u < 0) break;
            sm100::mbar_wait(&tfull[a], use & 1u);
            sm100::tc_fence_after();
            const uint32_t taddr = tmem + (quarter << 16) + (uint32_t)a * kBufCols;
            uint32_t v[2 * kNB];
#pragma unroll
            for (int i = 0; i < 2 * kNB; ++i) v[i] = sm100::tmem_ld_32x32b_x1(taddr + 16u * (uint32_t)i);
            sm100::tmem_wait_ld();
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tempty[a]);
#pragma unroll
            for (int i = 0; i < 2 * kNB; ++i) acc[i] += (double)__uint_as_float(v[i]);
            if (++k == prm.nk) {  // the unit's last stage: its segments are done
#pragma unroll
                for (int i = 0; i < 2 * kNB; ++i) {  // box i / 2, half i % 2
                    const size_t seg = ((size_t)u * kNB + (size_t)(i >> 1)) * kRtRows + (size_t)(i & 1) * 128u +
                                       (size_t)row;
                    if (seg < prm.S) out[seg] = (float)acc[i];
                    acc[i] = 0.0;
                }
                k = 0;
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc(tmem, kCols);
    // the last CTA resets the unit counter (every CTA's tickets precede its
    // completion ticket in thread 0's program order)
    if (prm.dyn && threadIdx.x == 0 && ticket_acq_rel(ws.ticket) == gridDim.x - 1) {
        *ws.chunk_next = 0u;
        *ws.ticket = 0u;
    }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                 CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                 CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiled>(p);
    }();
    return fn;
}

}  // namespace

// Applicability (checked by the caller): any element format, x 16-byte
// aligned, the row pitch L * element bytes a multiple of 16 (the tensor
// map's), S >= 1; rows and L below 2^31.
bool rows_tc05_supported(int fmt, const void* x, size_t S, size_t L) {
    const size_t lb = L * ((fmt == kE4M3 || fmt == kE5M2) ? 1 : 2);
    return fmt >= kF16 && fmt <= kE5M2 && ((uintptr_t)x & 15u) == 0 && lb % 16 == 0 && lb >= 16 &&
           L < ((size_t)1 << 31) && S >= 1 && S < ((size_t)1 << 31) - 4096 &&  // box rows fit int32
           encode_fn() != nullptr;
}

template <int BW, bool kF8>
static cudaError_t launch_rows_bw(EncodeTiled enc, int fmt, const void* x, size_t S, size_t L, float* out,
                                  const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream) {
    using Geo = RtGeom<BW>;
    constexpr size_t es = kF8 ? 1 : 2;  // element bytes
    constexpr int kBoxEl = BW * 2 / (int)es;  // elements per box row
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)S};
    const cuuint64_t strides[1] = {(cuuint64_t)(L * es)};
    const cuuint32_t box[2] = {(cuuint32_t)kBoxEl, (cuuint32_t)kRtRows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUtensorMapSwizzle sw = BW == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : BW == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
    if (enc(&map, kF8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(x),
            dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    RtParams prm;
    prm.S = S;
    prm.nk = (int)((L + kBoxEl - 1) / kBoxEl);
    prm.stages = cfg.rows_tc05_stages;
    // kind::f16: a/b format F16 = 0, BF16 = 1; kind::f8f6f4: E4M3 = 0, E5M2 = 1
    const uint32_t ab = (fmt == kBF16 || fmt == kE5M2) ? ((1u << 7) | (1u << 10)) : 0u;
    prm.idesc = sm100::idesc_f16_f32(128, 16) | ab;
    prm.one_bits = fmt == kBF16 ? 0x3F803F80u : fmt == kE4M3 ? 0x38383838u : fmt == kE5M2 ? 0x3C3C3C3Cu
                                                                                         : 0x3C003C00u;
    if (prm.stages < 2 ||
        kRtHeader - 8 < 512 + (size_t)(2 * prm.stages + 3 * kRtAcc) * 8 + (size_t)(prm.stages + kRtAcc) * 4)
        return cudaErrorInvalidValue;
    const size_t smem = kRtHeader + (size_t)prm.stages * kRtStageBytes;
    auto kernel = reduce_rows_tc05_kernel<BW, kF8>;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        static std::mutex mu;
        static std::map<int, size_t> configured;  // largest dynamic SMEM set so far, per device
        std::lock_guard<std::mutex> lk(mu);
        size_t& have = configured[dev];
        if (smem > have) {
            if ((e = cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem)))
                return e;
            have = smem;
        }
    }
    const size_t units = (S + (size_t)kRtRows * Geo::kNB - 1) / ((size_t)kRtRows * Geo::kNB);
    size_t g = (size_t)cfg.sms;
    if (g > units) g = units;
    // the dynamic tail (TCR_CFG_TC05_DYNAMIC percent of the units) when every
    // CTA has a run of at least 8 units
    prm.dyn = (units >= 8 * g) ? (long long)(units * (size_t)cfg.tc05_dynamic / 100u) : 0;
    launch_maybe_pdl(kernel, dim3((unsigned)g), dim3(kRtWarps * 32), smem, stream, cfg.pdl, map, prm, out, ws);
    return cudaGetLastError();
}

// Box width by segment bytes: 32 B (<= 32), 64 B (<= 64), else 128 B.
template <bool kF8>
static cudaError_t launch_rows_fmt(EncodeTiled enc, int fmt, const void* x, size_t S, size_t L, float* out,
                                   const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream) {
    const size_t lb = L * (kF8 ? 1 : 2);
    if (lb <= 32) return launch_rows_bw<16, kF8>(enc, fmt, x, S, L, out, ws, cfg, stream);
    if (lb <= 64) return launch_rows_bw<32, kF8>(enc, fmt, x, S, L, out, ws, cfg, stream);
    return launch_rows_bw<64, kF8>(enc, fmt, x, S, L, out, ws, cfg, stream);
}

cudaError_t launch_reduce_rows_tc05(int fmt, const void* x, size_t S, size_t L, float* out,
                                    const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    if (fmt == kE4M3 || fmt == kE5M2) return launch_rows_fmt<true>(enc, fmt, x, S, L, out, ws, cfg, stream);
    return launch_rows_fmt<false>(enc, fmt, x, S, L, out, ws, cfg, stream);
}

}  // namespace tcr
