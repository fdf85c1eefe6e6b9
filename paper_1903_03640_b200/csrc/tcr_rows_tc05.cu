// tcr_rows_tc05.cu -- fixed-length segments (tcr_reduce_sum_batched) on the
// 5th-generation tensor cores, 128 segments per MMA as the 128 rows of A:
//
//   HBM --(TMA tensor copy: 2-D map {L, S}, box {64 elements, 128 rows},
//   128-byte swizzle)--> 16 KiB SMEM stage in the canonical K-major SW128
//   layout --(4 x tcgen05.mma M128 N16 K16, the K slices at +32 B, B = ones)
//   --> one fp32 TMEM accumulator per box --(tcgen05.ld, one row per
//   thread)--> binary64 per segment --> out[j].
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
// warp % 4: rows 32 (warp % 4) .. + 31).  Row blocks are dealt to CTAs in
// grid-stride order; every role walks the same (block, box) sequence.
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
constexpr int kRtRows = 128;                     // segments per box = M
constexpr uint32_t kRtStageBytes = kRtBoxK * 2 * kRtRows;  // 16 KiB
constexpr uint32_t kRtHeader = 1024;             // ones tile + barriers + TMEM address
constexpr int kRtAcc = 4;                        // TMEM accumulators (16 columns each)
constexpr uint32_t kRtSlotCols = 16;

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
};

__global__ void __launch_bounds__(kRtWarps * 32)
reduce_rows_tc05_kernel(const __grid_constant__ CUtensorMap map, RtParams prm, float* __restrict__ out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int stages = prm.stages;
    uint32_t* ones = reinterpret_cast<uint32_t*>(smem);        // 512 B of ones (B operand)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 512);  // [stages]
    uint64_t* empty = full + stages;                           // [stages]
    uint64_t* tfull = empty + stages;                          // [kRtAcc]
    uint64_t* tempty = tfull + kRtAcc;                         // [kRtAcc]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kRtHeader - 8);
    uint8_t* ring = smem + kRtHeader;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const size_t blocks = (prm.S + kRtRows - 1) / kRtRows;
    const size_t G = gridDim.x, b0 = blockIdx.x;
    const long long my_blocks = b0 < blocks ? (long long)((blocks - b0 + G - 1) / G) : 0;
    const long long boxes = my_blocks * prm.nk;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < kRtAcc; ++a) {
            sm100::mbar_init(&tfull[a], 1);
            sm100::mbar_init(&tempty[a], 4);
        }
        sm100::fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    }
    for (int i = threadIdx.x; i < 128; i += blockDim.x) ones[i] = prm.one_bits;
    sm100::fence_proxy_async_smem();
    constexpr uint32_t kCols = kRtAcc * kRtSlotCols;  // 64 columns
    if (warp == 1) sm100::tmem_alloc(tmem_slot, kCols);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait_and_release();  // the previous kernel's writes (x, out) visible

    if (warp == 0) {
        if (lane == 0) {  // producer: one TMA box per (row block, K box)
            int s = 0;
            uint32_t ph = 0;
            for (long long j = 0; j < boxes; ++j) {
                const long long u = (long long)b0 + (j / prm.nk) * (long long)G;
                const int k = (int)(j % prm.nk);
                sm100::mbar_wait(&empty[s], ph ^ 1u);
                sm100::mbar_arrive_expect_tx(&full[s], kRtStageBytes);
                tma_load_2d(ring + (size_t)s * kRtStageBytes, &map, k * kRtBoxK, (int)(u * kRtRows), &full[s]);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer: 4 MMAs per box into accumulator j % kRtAcc
            const uint64_t bdesc = sm100::smem_desc_kmajor(sm100::smem_addr(ones), 128, 256);
            const uint64_t adesc0 = smem_desc_sw128(sm100::smem_addr(ring));
            constexpr uint64_t kStageStep = kRtStageBytes >> 4;
            int s = 0;
            uint32_t ph = 0;
            for (long long j = 0; j < boxes; ++j) {
                const int a = (int)(j % kRtAcc);
                const uint32_t use = (uint32_t)(j / kRtAcc);
                sm100::mbar_wait(&full[s], ph);
                sm100::mbar_wait(&tempty[a], (use & 1u) ^ 1u);  // drained kRtAcc boxes ago
                sm100::tc_fence_after();
                const uint64_t ad = adesc0 + (uint64_t)s * kStageStep;
                const uint32_t d = tmem + (uint32_t)a * kRtSlotCols;
#pragma unroll
                for (int q = 0; q < kRtBoxK / 16; ++q)  // K slice q: +32 B = +2 in the descriptor
                    sm100::mma_f16_ss(d, ad + (uint64_t)(2 * q), bdesc, prm.idesc, q > 0 ? 1u : 0u);
                sm100::mma_commit(&tfull[a]);
                sm100::mma_commit(&empty[s]);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        __syncwarp();
    } else {  // epilogue: row r = 32 (warp % 4) + lane of every box
        const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
        const int row = (int)quarter + lane;
        double acc = 0.0;
        for (long long j = 0; j < boxes; ++j) {
            const int a = (int)(j % kRtAcc);
            const uint32_t use = (uint32_t)(j / kRtAcc);
            sm100::mbar_wait(&tfull[a], use & 1u);
            sm100::tc_fence_after();
            const uint32_t v = sm100::tmem_ld_32x32b_x1(tmem + (quarter << 16) + (uint32_t)a * kRtSlotCols);
            sm100::tmem_wait_ld();
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tempty[a]);
            acc += (double)__uint_as_float(v);
            if ((int)(j % prm.nk) == prm.nk - 1) {  // the row block's last box: segment done
                const size_t u = b0 + (size_t)(j / prm.nk) * G;
                const size_t seg = u * kRtRows + (size_t)row;
                if (seg < prm.S) out[seg] = (float)acc;
                acc = 0.0;
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc(tmem, kCols);
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
                                    const LaunchCfg& cfg, cudaStream_t stream) {
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
    if (prm.stages < 2 || kRtHeader - 8 < 512 + (size_t)(2 * prm.stages + 2 * kRtAcc) * 8)
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
    launch_maybe_pdl(reduce_rows_tc05_kernel, dim3((unsigned)g), dim3(kRtWarps * 32), smem, stream, cfg.pdl,
                     map, prm, out);
    return cudaGetLastError();
}

}  // namespace tcr
