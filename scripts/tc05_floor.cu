// tc05_floor.cu -- diagnostic (not part of libtcr): the floor of the
// single-thread tcgen05.mma issue cost on B200 (r02), to tell the hardware
// cost from the cost of per-MMA descriptor arithmetic:
//   mode 0: the same A / B descriptors and D address for every MMA
//   mode 1: 16 MMAs per group fully unrolled, A = base + compile-time
//           constant offset (ptxas can fold the offsets)
//   mode 2: A computed per MMA from the loop counter (as the library does)
// M = 128, N = 16 (input as A, 4 KiB per MMA), kind::f16; commit every 16
// MMAs, 4 groups in flight (one mbarrier per group slot), 1 CTA per SM on all
// SMs; bounded waits (a diagnostic never hangs the GPU).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1903_03640_b200/csrc/tcr_sm100.cuh"

using namespace tcr::sm100;

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ bool g_timed_out = false;
__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
    const unsigned long long t0 = now();
    while (!mbar_try_wait(bar, parity))
        if (now() - t0 > 20000000ull) { g_timed_out = true; return; }
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) floor_k(int groups, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [4]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 64);
    uint8_t* in = smem + 1024;            // 64 KiB: 16 A tiles of 4 KiB
    uint8_t* ones = smem + 1024 + 65536;  // 512 B
    for (int i = threadIdx.x; i < (65536 + 512) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(in)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int b = 0; b < 4; ++b) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc(tslot, 64);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_f16_f32(128, 16);
        const uint64_t bd = smem_desc_kmajor(smem_addr(ones), 128, 256);
        const uint64_t a0 = smem_desc_kmajor(smem_addr(in), 128, 256);
        uint32_t ph[4] = {0u, 0u, 0u, 0u};
        const unsigned long long t0 = now();
        for (int g = 0; g < groups; ++g) {
            const int b = g & 3;
            if (g >= 4) { wait_bounded(&bars[b], ph[b]); ph[b] ^= 1u; }
            if constexpr (MODE == 0) {
#pragma unroll
                for (int k = 0; k < 16; ++k) mma_f16_ss(tmem, a0, bd, idesc, 1u);
            } else if constexpr (MODE == 1) {
#pragma unroll
                for (int k = 0; k < 16; ++k) mma_f16_ss(tmem + (k & 3) * 16, a0 + (uint64_t)(k * 256), bd, idesc, 1u);
            } else {
                for (int k = 0; k < 16; ++k) {
                    const int j = g * 16 + k;
                    mma_f16_ss(tmem + (uint32_t)((j & 3) * 16), a0 + (uint64_t)((j & 15) * 256), bd, idesc, 1u);
                }
            }
            mma_commit(&bars[b]);
        }
        for (int g = groups > 4 ? groups - 4 : 0; g < groups; ++g) {
            wait_bounded(&bars[g & 3], ph[g & 3]);
            ph[g & 3] ^= 1u;
        }
        out[blockIdx.x] = now() - t0;
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 64);
}

template <int MODE>
static void run(int sms, unsigned long long* out, const char* name) {
    const size_t smem = 1024 + 65536 + 1024;
    cudaFuncSetAttribute(floor_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int groups = 1000;
    floor_k<MODE><<<sms, 128, smem>>>(groups, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("%s error %s\n", name, cudaGetErrorString(e)); fflush(stdout); return; }
    bool to = false;
    cudaMemcpyFromSymbol(&to, g_timed_out, sizeof(bool));
    unsigned long long h[256];
    cudaMemcpy(h, out, 8 * sms, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double ns = (double)mx / (16.0 * groups);
    printf("%-44s %6.1f ns/MMA  %6.1f GB/s/SM  %6.0f GB/s chip%s\n", name, ns, 4096.0 / ns,
           4096.0 / ns * sms, to ? "  TIMED OUT" : "");
    fflush(stdout);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out;
    cudaMalloc(&out, 8 * 256);
    for (int r = 0; r < 2; ++r) {
        run<0>(sms, out, "mode 0: constant descriptors, one D");
        run<1>(sms, out, "mode 1: unrolled, constant offsets, 4 D");
        run<2>(sms, out, "mode 2: descriptors from the loop counter");
    }
    return 0;
}
