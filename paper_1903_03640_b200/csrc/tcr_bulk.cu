// tcr_bulk.cu -- the MMA-encoded reduction fed through shared memory by the
// TMA engine (the north star's "128-bit loads staged through shared memory"):
//
//   HBM --(cp.async.bulk, one elected producer lane)--> SMEM ring of
//   `stages` x `stage_kb` KiB --(ld.shared.v4 by 8 consumer warps)--> mma.sync
//   m16n8k16 D = A x 1 + C (Eq. 9-10) --> fp64 lane accumulators --> the
//   shared warp / CTA / grid completion (D' = 1 x D, Eq. 11-12).
//
// Bytes in flight per SM are bounded by shared memory (up to ~200 KiB), not by
// registers, and no single thread issues the tensor work (the limit of the
// tcgen05 path at N = 16, profiles/r01/tc05_issue.txt).  Each 512-byte tile
// of a stage is one consumer lane-vector per lane, consumed by warp
// (tile % 8); every 4 KiB of a 16 KiB stage therefore feeds a different
// warp, and each warp carries its fp32 chain over 2 tiles per accumulator per
// stage before flushing to fp64 (K = 2 x stages-per-flush).
#include <map>
#include <mutex>

#include "tcr_complete.cuh"
#include "tcr_device.cuh"
#include "tcr_internal.h"
#include "tcr_sm100.cuh"

namespace tcr {

namespace {

constexpr int kConsumers = 8;                 // consumer warps
constexpr int kBulkWarps = kConsumers + 1;    // + producer warp
constexpr uint32_t kBulkHeader = 1024;        // barriers

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(sm100::smem_addr(p)));
    return r;
}

}  // namespace

template <int F>
__global__ void __launch_bounds__(kBulkWarps * 32)
reduce_bulk_kernel(const uint8_t* __restrict__ x, size_t n, int stages, uint32_t stage_bytes,
                   int flush_every, float* out_f32, double* out_f64, DevWorkspace ws) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + stages;
    uint8_t* ring = smem + kBulkHeader;
    constexpr int ES = FmtInfo<F>::kBytes;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const size_t nbytes = n * ES;
    size_t head = (16u - ((uintptr_t)x & 15u)) & 15u;
    if (head > nbytes) head = nbytes;
    const uint8_t* xa = x + head;
    const size_t nb = nbytes - head;
    const size_t C = nb / stage_bytes;
    const size_t G = gridDim.x, b = blockIdx.x;
    const size_t c_begin = b * C / G;
    const int nchunks = (int)((b + 1) * C / G - c_begin);
    const int tiles = (int)(stage_bytes / 512);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], kConsumers);
        }
        sm100::fence_mbar_init();
    }
    __syncthreads();
    pdl_wait_and_release();  // PDL: no global memory before the previous kernel completes

    double acc = 0.0;
    if (warp == kConsumers) {  // producer warp
        if (lane == 0 && nchunks > 0) {
            const uint64_t pol = sm100::policy_evict_first();
            const uint8_t* src = xa + c_begin * (size_t)stage_bytes;
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nchunks; ++i, src += stage_bytes) {
                sm100::mbar_wait(&empty[s], ph ^ 1u);
                sm100::mbar_arrive_expect_tx(&full[s], stage_bytes);
                sm100::bulk_g2s(ring + (size_t)s * stage_bytes, src, stage_bytes, &full[s], pol);
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        __syncwarp();
    } else {  // consumer warps
        float cA[4] = {0.f, 0.f, 0.f, 0.f}, cB[4] = {0.f, 0.f, 0.f, 0.f};
        int s = 0, it = 0;
        uint32_t ph = 0;
        for (int i = 0; i < nchunks; ++i) {
            sm100::mbar_wait(&full[s], ph);
            const uint8_t* stage = ring + (size_t)s * stage_bytes + lane * 16;
            int k = 0;
            for (int t = warp; t < tiles; t += kConsumers, ++k) {
                const uint4 v = lds128(stage + (size_t)t * 512);
                if (k & 1) mma_rowsum_f<F>(cB, v);
                else mma_rowsum_f<F>(cA, v);
            }
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&empty[s]);  // stage consumed by this warp
            if (++it == flush_every) {
                it = 0;
                flush_rows(cA, acc, lane);
                flush_rows(cB, acc, lane);
            }
            if (++s == stages) {
                s = 0;
                ph ^= 1u;
            }
        }
        flush_rows(cA, acc, lane);
        flush_rows(cB, acc, lane);
        if (blockIdx.x == gridDim.x - 1) {
            // ragged work past the last full chunk, and the unaligned head
            const uint8_t* xr = xa + C * (size_t)stage_bytes;
            const size_t rem = nb - C * (size_t)stage_bytes;
            const size_t Tr = rem / 512;
            const int tail = (int)(rem - Tr * 512);
            const uint4* base = reinterpret_cast<const uint4*>(xr) + lane;
            float c[4] = {0.f, 0.f, 0.f, 0.f};
            for (size_t t = warp; t < Tr; t += kConsumers) {
                mma_rowsum_f<F>(c, ldg_stream(base + t * 32));
                flush_rows(c, acc, lane);
            }
            if (warp == 0 && head) {
                mma_rowsum_f<F>(c, load_ragged_bytes(x, (int)head, lane));
                flush_rows(c, acc, lane);
            }
            if (warp == 1 && tail) {
                mma_rowsum_f<F>(c, load_ragged_bytes(xr + Tr * 512, tail, lane));
                flush_rows(c, acc, lane);
            }
        }
    }
    complete_block_and_grid<true, kBulkWarps>(acc, out_f32, out_f64, ws);
}

static int bulk_resident(const LaunchCfg& cfg) {
    const size_t smem = kBulkHeader + (size_t)cfg.bulk_stages * cfg.bulk_stage_kb * 1024u;
    int r = cfg.bulk_ctas < 1 ? 1 : cfg.bulk_ctas;
    const int by_smem = (int)((227u * 1024u) / smem);
    if (r > by_smem) r = by_smem;
    return r < 1 ? 1 : r;
}

template <int F>
static cudaError_t launch_bulk_t(const uint8_t* x, size_t n, float* out_f32, double* out_f64,
                                 const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream) {
    const int stages = cfg.bulk_stages;
    const uint32_t stage_bytes = (uint32_t)cfg.bulk_stage_kb * 1024u;
    if (stages < 2 || stages > 32 || stage_bytes < 4096 || stage_bytes % 4096 ||
        kBulkHeader < (size_t)2 * stages * 8)
        return cudaErrorInvalidValue;
    const size_t smem = kBulkHeader + (size_t)stages * stage_bytes;
    if (smem > 227u * 1024u) return cudaErrorInvalidValue;  // one CTA's shared memory limit
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        static std::mutex mu;
        static std::map<int, size_t> configured;
        std::lock_guard<std::mutex> lk(mu);
        if (smem > configured[dev]) {
            if ((e = cudaFuncSetAttribute(reduce_bulk_kernel<F>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
                return e;
            configured[dev] = smem;
        }
    }
    const size_t C = n * FmtInfo<F>::kBytes / stage_bytes;
    size_t g = (size_t)cfg.sms * bulk_resident(cfg);
    if (g > C) g = C;
    if (g < 1) g = 1;
    // chain K = 2 tiles per accumulator per stage (16 KiB stage, 8 warps) x flush_every
    const int tiles_per_warp = (int)(stage_bytes / 512 / kConsumers);
    int fe = 2 * cfg.chain / (tiles_per_warp < 1 ? 1 : tiles_per_warp);
    if (fe < 1) fe = 1;
    launch_maybe_pdl(reduce_bulk_kernel<F>, dim3((unsigned)g), dim3(kBulkWarps * 32), smem, stream, cfg.pdl,
                     x, n, stages, stage_bytes, fe, out_f32, out_f64, ws);
    return cudaGetLastError();
}

cudaError_t launch_reduce_bulk(int fmt, const uint16_t* x16, size_t n, float* out_f32,
                               double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                               cudaStream_t stream) {
    const uint8_t* x = reinterpret_cast<const uint8_t*>(x16);
    switch (fmt) {
        case kBF16: return launch_bulk_t<kBF16>(x, n, out_f32, out_f64, ws, cfg, stream);
        case kE4M3: return launch_bulk_t<kE4M3>(x, n, out_f32, out_f64, ws, cfg, stream);
        case kE5M2: return launch_bulk_t<kE5M2>(x, n, out_f32, out_f64, ws, cfg, stream);
        default: return launch_bulk_t<kF16>(x, n, out_f32, out_f64, ws, cfg, stream);
    }
}

}  // namespace tcr
