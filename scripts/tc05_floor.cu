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
//   mode 3: mode 2 + a second commit per group (the library commits per SMEM
//           stage AND per accumulator round)
//   mode 4: mode 2 with the library's accumulate pattern (first MMA of each
//           of the 4 accumulators per group overwrites)
//   mode 5: mode 2 while warp 1 streams cp.async.bulk 16 KiB copies from HBM
//           into a separate SMEM region (TMA writes competing for SMEM)
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
__global__ void __launch_bounds__(128, 1) floor_k(int groups, unsigned long long* out,
                                                  const uint8_t* src, size_t src_bytes) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [4] + [4] second commits + [2] tma
    uint64_t* bars2 = bars + 4;
    uint64_t* tbar = bars + 8;
    volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(smem + 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 64);
    uint8_t* in = smem + 1024;            // 64 KiB: 16 A tiles of 4 KiB
    uint8_t* ones = smem + 1024 + 65536;  // 512 B
    uint8_t* tbuf = smem + 1024 + 65536 + 1024;  // 2 x 16 KiB TMA landing zone (mode 5)
    for (int i = threadIdx.x; i < (65536 + 512) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(in)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int b = 0; b < 10; ++b) mbar_init(&bars[b], 1);
        *stop = 0u;
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
            if constexpr (MODE >= 3) {
                for (int k = 0; k < 16; ++k) {
                    const int j = g * 16 + k;
                    const uint32_t acc = (MODE == 4 && k < 4) ? 0u : 1u;
                    mma_f16_ss(tmem + (uint32_t)((j & 3) * 16), a0 + (uint64_t)((j & 15) * 256), bd, idesc, acc);
                }
                if constexpr (MODE == 3) mma_commit(&bars2[b]);
            } else if constexpr (MODE == 0) {
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
        *stop = 1u;
    } else if (MODE == 5 && threadIdx.x == 32) {  // TMA streamer: 2 x 16 KiB, until stopped
        const size_t per = src_bytes / gridDim.x / 16384 * 16384;
        const uint8_t* base = src + (size_t)blockIdx.x * per;
        uint32_t tph[2] = {0u, 0u};
        size_t off = 0;
        for (int i = 0; !*stop; ++i) {
            const int b = i & 1;
            if (i >= 2) { wait_bounded(&tbar[b], tph[b]); tph[b] ^= 1u; }
            mbar_arrive_expect_tx(&tbar[b], 16384);
            bulk_g2s(tbuf + b * 16384, base + off, 16384, &tbar[b], policy_evict_first());
            off += 16384;
            if (off >= per) off = 0;
        }
        for (int b = 0; b < 2; ++b) wait_bounded(&tbar[b], tph[b]);
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 64);
}

template <int MODE>
static void run(int sms, unsigned long long* out, const char* name, const uint8_t* src, size_t sb) {
    const size_t smem = 1024 + 65536 + 1024 + 32768;
    cudaFuncSetAttribute(floor_k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int groups = 1000;
    floor_k<MODE><<<sms, 128, smem>>>(groups, out, src, sb);
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
    const size_t sb = (size_t)1 << 30;
    uint8_t* src;
    cudaMalloc(&src, sb);
    cudaMemset(src, 1, sb);
    for (int r = 0; r < 2; ++r) {
        run<0>(sms, out, "mode 0: constant descriptors, one D", src, sb);
        run<1>(sms, out, "mode 1: unrolled, constant offsets, 4 D", src, sb);
        run<2>(sms, out, "mode 2: descriptors from the loop counter", src, sb);
        run<3>(sms, out, "mode 3: + a second commit per group", src, sb);
        run<4>(sms, out, "mode 4: + library accumulate pattern", src, sb);
        run<5>(sms, out, "mode 5: mode 2 + concurrent TMA into SMEM", src, sb);
    }
    return 0;
}
