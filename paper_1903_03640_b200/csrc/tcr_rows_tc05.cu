// tcr_rows_tc05.cu -- fixed-length segments (tcr_reduce_sum_batched) on the
// 5th-generation tensor cores, 128 segments per MMA as the 128 rows of A:
//
//   HBM --(TMA tensor copy: 2-D map {L, S}, box {64 elements, 256 rows},
//   128-byte swizzle)--> 32 KiB SMEM stage in the canonical K-major SW128
//   layout --(2 x 4 tcgen05.mma M128 N16 K16: the box's two 128-row halves,
//   the K slices at +32 B, B = ones)--> two fp32 TMEM accumulators per box
//   --(tcgen05.ld, two rows per thread)--> binary64 per segment --> out[j].
//
// Paper mapping (arXiv 1903.03640): D = A x 1 (Eq. 9-10) with row
// r of A holding 64 elements of segment r: "the m row sums" are the segment
// partial sums directly, so no D' = 1 x D collapse per segment is needed --
// the collapse that recombines one group's row sums (Eq. 11-12) has nothing
// to do when every row is a different segment.  A box's 4 MMAs are the
// carried chain (K = 4, reading G9); each box's row sums are flushed into
// binary64 (bounded truncation, reading G10).  A segment's boxes are added in
// index order by one thread: deterministic, independent of the grid.
//
// The tensor map's out-of-bounds fill supplies the paper's zero padding of
// the trailing group (reading G5): boxes past L (L not a multiple of 64) and
// rows past S (S not a multiple of 128) arrive as zeros.
//
// Warp roles (192 threads): warp 0 lane 0 producer (TMA), warp 1 lane 0 MMA
// issuer (warp 1 allocates TMEM), warps 2-5 epilogue (TMEM lane quarter
// warp % 4: rows 32 (warp % 4) .. + 31 of both halves).  256-row boxes (32
// KiB, 8 MMAs) rather than 128-row ones: the issuing thread's per-box
// bookkeeping (two barrier waits, a commit pair, the block hand-off) was the
// limit at 16 KiB per box.
#include <cuda.h>

#include <map>
#include <mutex>

#include "tcr_device.cuh"
#include "tcr_internal.h"
#include "tcr_sm100.cuh"

namespace tcr {

namespace {

constexpr int kRtWarps = 6;
constexpr int kRtBoxK = 64;                      // elements of a segment per box (128 B)
constexpr int kRtRows = 256;                     // segments per box = 2 x M
constexpr uint32_t kRtHalfBytes = kRtBoxK * 2 * 128;       // one M = 128 half: 16 KiB
constexpr uint32_t kRtStageBytes = 2 * kRtHalfBytes;       // 32 KiB
constexpr uint32_t kRtHeader = 1024;             // ones tile + barriers + TMEM address
constexpr int kRtAcc = 4;                        // TMEM accumulator pairs (2 x 16 columns each)
constexpr uint32_t kRtSlotCols = 32;

// K-major, 128-byte-swizzle UMMA descriptor of a 128 x 64 (16-bit) SMEM tile
// written by a SWIZZLE_128B TMA box: 8-row atoms of 1024 B (SBO), rows of
// 128 B inside an atom, the XOR swizzle applied by the hardware on address
// bits; LBO unused (1); version 1 (sm_100); layout type 2 = SWIZZLE_128B.
// The K slice k (16 elements = 32 B) starts 32 k bytes into the tile.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;                  // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024u >> 4) << 32;       // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
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
    int nk;          // boxes per row block = ceil(L / 64)
    int stages;      // SMEM ring stages
    uint32_t idesc;  // kind::f16 instruction descriptor (F16 or BF16 operands)
    uint32_t one_bits;
    long long dyn;   // row blocks handed out by ticket at the end (the dynamic tail)
};

// Row blocks [0, Bs) are dealt in grid-stride order, the last `dyn` blocks
// one at a time from ws.chunk_next
// (two tickets held ahead), as the flat kernel's dynamic tail (§16): every
// block is reduced by one CTA in box order, so the schedule cannot change a
// bit.  The producer writes each stage's block index (-1 = END) next to the
// stage; the MMA issuer forwards it per accumulator with a plain arrive on
// tinf[a] (release), which the epilogue waits on before reading it.
__global__ void __launch_bounds__(kRtWarps * 32)
reduce_rows_tc05_kernel(const __grid_constant__ CUtensorMap map, RtParams prm, float* __restrict__ out,
                        DevWorkspace ws) {
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

    const long long blocks = (long long)((prm.S + kRtRows - 1) / kRtRows);
    const long long Bs = blocks - prm.dyn;
    const long long G = gridDim.x, b = blockIdx.x;
    // static part in grid-stride order (CTA b: blocks b, b + G, ... < Bs): at
    // any moment the grid reads neighbouring blocks (contiguous runs per CTA
    // measured ~10 % slower, profiles/r02/rows_tc05_ab2.txt)
    const long long n_static = b < Bs ? (Bs - b + G - 1) / G : 0;

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
    constexpr uint32_t kCols = kRtAcc * kRtSlotCols;  // 128 columns
    if (warp == 1) sm100::tmem_alloc(tmem_slot, kCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait_and_release();  // the previous kernel's writes (x, out, counters) visible

    if (warp == 0) {
        if (lane == 0) {  // producer: nk TMA boxes per row block, then END
            int s = 0;
            uint32_t ph = 0;
            auto block_boxes = [&](long long u) {
                for (int k = 0; k < prm.nk; ++k) {
                    sm100::mbar_wait(&empty[s], ph ^ 1u);
                    sinfo[s] = (int)u;
                    sm100::mbar_arrive_expect_tx(&full[s], kRtStageBytes);
                    tma_load_2d(ring + (size_t)s * kRtStageBytes, &map, k * kRtBoxK, (int)(u * kRtRows),
                                &full[s]);
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
                block_boxes(b + i * G);
            }
            if (prm.dyn) {
                if (!f0) t0 = atomicAdd(ws.chunk_next, 1u);
                if (!f1) t1 = atomicAdd(ws.chunk_next, 1u);
                for (;;) {
                    const unsigned t = t0;
                    t0 = t1;
                    t1 = atomicAdd(ws.chunk_next, 1u);
                    if ((long long)t >= prm.dyn) break;
                    block_boxes(Bs + (long long)t);
                }
            }
            sm100::mbar_wait(&empty[s], ph ^ 1u);  // END: a stage with no bytes
            sinfo[s] = -1;
            sm100::mbar_arrive(&full[s]);
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer: 2 x 4 MMAs per box into accumulator pair j % kRtAcc
            const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
            const uint64_t adesc0 = smem_desc_sw128(sm100::smem_addr(ring));
            constexpr uint64_t kStageStep = kRtStageBytes >> 4;
            int s = 0;
            uint32_t ph = 0;
            for (long long j = 0;; ++j) {
                const int a = (int)(j % kRtAcc);
                const uint32_t use = (uint32_t)(j / kRtAcc);
                sm100::mbar_wait(&full[s], ph);
                const int u = sinfo[s];
                sm100::mbar_wait(&tempty[a], (use & 1u) ^ 1u);  // drained kRtAcc boxes ago
                tinfo[a] = u;
                if (u < 0) {
                    sm100::mbar_arrive(&tinf[a]);
                    break;
                }
                sm100::tc_fence_after();
                const uint64_t ad = adesc0 + (uint64_t)s * kStageStep;
                const uint32_t d = tmem + (uint32_t)a * kRtSlotCols;
#pragma unroll
                for (int h = 0; h < 2; ++h)  // rows 128 h .. 128 h + 127 of the box: +16 KiB
#pragma unroll
                    for (int q = 0; q < kRtBoxK / 16; ++q)  // K slice q: +32 B = +2 in the descriptor
                        sm100::mma_f16_ss(d + 16u * (uint32_t)h, ad + (uint64_t)(h * (kRtHalfBytes >> 4) + 2 * q),
                                          bdesc, prm.idesc, q > 0 ? 1u : 0u);
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
    } else {  // epilogue: row r = 32 (warp % 4) + lane of every box
        const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
        const int row = (int)quarter + lane;  // and row + 128 (the box's second M half)
        double acc = 0.0, acc2 = 0.0;
        int k = 0;
        for (long long j = 0;; ++j) {
            const int a = (int)(j % kRtAcc);
            const uint32_t use = (uint32_t)(j / kRtAcc);
            sm100::mbar_wait(&tinf[a], use & 1u);
            const int u = tinfo[a];
            if (u < 0) break;
            sm100::mbar_wait(&tfull[a], use & 1u);
            sm100::tc_fence_after();
            const uint32_t taddr = tmem + (quarter << 16) + (uint32_t)a * kRtSlotCols;
            const uint32_t v = sm100::tmem_ld_32x32b_x1(taddr);
            const uint32_t v2 = sm100::tmem_ld_32x32b_x1(taddr + 16u);
            sm100::tmem_wait_ld();
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tempty[a]);
            acc += (double)__uint_as_float(v);
            acc2 += (double)__uint_as_float(v2);
            if (++k == prm.nk) {  // the row block's last box: its segments are done
                const size_t seg = (size_t)u * kRtRows + (size_t)row;
                if (seg < prm.S) out[seg] = (float)acc;
                if (seg + 128 < prm.S) out[seg + 128] = (float)acc2;
                acc = acc2 = 0.0;
                k = 0;
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc(tmem, kCols);
    // the last CTA resets the block counter (every CTA's tickets precede its
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

// Applicability (checked by the caller): binary16 / bfloat16, x 16-byte
// aligned, L % 8 == 0 (the tensor map's row pitch must be a multiple of 16
// bytes), 8 <= L, S >= 1; rows and L below 2^31.
bool rows_tc05_supported(int fmt, const void* x, size_t S, size_t L) {
    return (fmt == kF16 || fmt == kBF16) && ((uintptr_t)x & 15u) == 0 && L % 8 == 0 && L >= 8 &&
           L < ((size_t)1 << 31) && S >= 1 && S < ((size_t)1 << 31) && encode_fn() != nullptr;
}

cudaError_t launch_reduce_rows_tc05(int fmt, const void* x, size_t S, size_t L, float* out,
                                    const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream) {
    EncodeTiled enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)S};
    const cuuint64_t strides[1] = {(cuuint64_t)L * 2u};
    const cuuint32_t box[2] = {(cuuint32_t)kRtBoxK, (cuuint32_t)kRtRows};
    const cuuint32_t estr[2] = {1u, 1u};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    RtParams prm;
    prm.S = S;
    prm.nk = (int)((L + kRtBoxK - 1) / kRtBoxK);
    prm.stages = cfg.rows_tc05_stages;
    const uint32_t ab = fmt == kBF16 ? ((1u << 7) | (1u << 10)) : 0u;
    prm.idesc = sm100::idesc_f16_f32(128, 16) | ab;
    prm.one_bits = fmt == kBF16 ? 0x3F803F80u : 0x3C003C00u;
    if (prm.stages < 2 ||
        kRtHeader - 8 < 512 + (size_t)(2 * prm.stages + 3 * kRtAcc) * 8 + (size_t)(prm.stages + kRtAcc) * 4)
        return cudaErrorInvalidValue;
    const size_t smem = kRtHeader + (size_t)prm.stages * kRtStageBytes;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        static std::mutex mu;
        static std::map<int, size_t> configured;  // largest dynamic SMEM set so far, per device
        std::lock_guard<std::mutex> lk(mu);
        size_t& have = configured[dev];
        if (smem > have) {
            if ((e = cudaFuncSetAttribute((const void*)reduce_rows_tc05_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
                return e;
            have = smem;
        }
    }
    const size_t blocks = (S + kRtRows - 1) / kRtRows;
    size_t g = (size_t)cfg.sms;
    if (g > blocks) g = blocks;
    // the dynamic tail (TCR_CFG_TC05_DYNAMIC percent of the row blocks) when
    // every CTA has a run of at least 8 blocks
    prm.dyn = (blocks >= 8 * g) ? (long long)(blocks * (size_t)cfg.tc05_dynamic / 100u) : 0;
    launch_maybe_pdl(reduce_rows_tc05_kernel, dim3((unsigned)g), dim3(kRtWarps * 32), smem, stream, cfg.pdl,
                     map, prm, out, ws);
    return cudaGetLastError();
}

}  // namespace tcr
