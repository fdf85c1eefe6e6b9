// tc05_micro.cu -- diagnostic microbenchmarks (not part of libtcr) that
// separate the two halves of the tcgen05 reduction pipeline on B200:
//   A) tcgen05.mma issue/throughput from SMEM for M=128, N in {16,32,64,256}
//      with 1 or 16 independent accumulators, one issuing thread per SM;
//   B) cp.async.bulk (TMA engine) global->shared throughput for a ring of
//      `stages` x `kb` KiB with an immediate-release consumer (no MMA).
// Prints cycles per MMA and GB/s.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o scripts/tc05_micro scripts/tc05_micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1903_03640_b200/csrc/tcr_sm100.cuh"

using namespace tcr::sm100;

__global__ void __launch_bounds__(128, 1) mma_rate(int iters, int slots, int N, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 8);
    uint8_t* a = smem + 1024;            // 64 KiB of A tiles
    uint8_t* b = smem + 1024 + 65536;    // B (N x 16 fp16, <= 8 KiB)
    for (int i = threadIdx.x; i < (65536 + 8192) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(a)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(tslot, 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_f16_f32(128, N);
        const uint64_t bdesc = smem_desc_kmajor(smem_addr(b), 128, 256);
        const uint64_t a0 = smem_desc_kmajor(smem_addr(a), 128, 256);
        const uint32_t stride = (uint32_t)N;  // columns per accumulator
        long long t0 = clock64();
        int s = 0;
        for (int i = 0; i < iters; ++i) {
            mma_f16_ss(tmem + (uint32_t)s * stride, a0 + (uint64_t)((i & 15) * 256), bdesc, idesc, 1u);
            if (++s == slots) s = 0;
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

__global__ void __launch_bounds__(64, 1) tma_rate(const uint8_t* src, size_t bytes_per_cta, int stages,
                                                  uint32_t stage_bytes) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + stages;
    uint8_t* ring = smem + 1024;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_mbar_init();
    }
    __syncthreads();
    const uint8_t* base = src + blockIdx.x * bytes_per_cta;
    const int n = (int)(bytes_per_cta / stage_bytes);
    if (threadIdx.x == 0) {
        const uint64_t pol = policy_evict_first();
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < n; ++i) {
            mbar_wait(&empty[s], ph ^ 1u);
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            bulk_g2s(ring + (size_t)s * stage_bytes, base + (size_t)i * stage_bytes, stage_bytes, &full[s], pol);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
    } else if (threadIdx.x == 32) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < n; ++i) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
    }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc; cudaMalloc(&cyc, sizeof(long long) * sms);
    cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 65536 + 8192);
    for (int N : {16, 32, 64, 256}) {
        for (int slots : {1, 4, 16}) {
            if (slots * N > 512) continue;
            const int iters = 4096;
            mma_rate<<<sms, 128, 1024 + 65536 + 8192>>>(iters, slots, N, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("mma_rate error %s\n", cudaGetErrorString(e)); return 1; }
            long long h[256]; cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("MMA M=128 N=%3d slots=%2d: %.1f cycles/MMA (max over SMs), %.1f elems/cycle/SM\n",
                   N, slots, (double)mx / iters, 2048.0 * iters / mx);
        }
    }
    const size_t bytes = (size_t)2 << 30;
    uint8_t* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
    cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 200 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int ctas : {1, 2}) {
        for (int kb : {4, 8, 16, 32, 64}) {
            for (int stages : {2, 4, 8, 12}) {
                const uint32_t sb = kb * 1024;
                const size_t smem = 1024 + (size_t)stages * sb;
                if (smem * ctas > 227 * 1024) continue;
                const int grid = sms * ctas;
                const size_t per = (bytes / grid) / sb * sb;
                float best = 1e30f;
                for (int r = 0; r < 6; ++r) {
                    cudaEventRecord(a);
                    tma_rate<<<grid, 64, smem>>>(src, per, stages, sb);
                    cudaEventRecord(b); cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b);
                    if (r && ms < best) best = ms;
                }
                cudaError_t e = cudaGetLastError();
                if (e) { printf("tma_rate error %s\n", cudaGetErrorString(e)); return 1; }
                printf("TMA bulk ctas/SM=%d stage=%2d KiB x %2d: %.1f GB/s\n", ctas, kb, stages,
                       per * grid / (best * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
