// tc05_pair.cu -- diagnostic (not part of libtcr): is a CTA pair
// (tcgen05.mma.cta_group::2, M = 256 across two SMs) a faster way to issue
// the reduction's A x ones MMAs than one CTA per SM (cta_group::1, M = 128)?
//
// The reduction's B is a constant ones tile and its A is never shared, so a
// pair only helps if one M = 256 instruction costs the issuing thread about
// what one M = 128 instruction costs (it then covers 2 x 4 KiB per issue
// slot).  Measured here: issuing-thread nanoseconds per group of 4 MMAs,
//   mode 0: cta_group::1, M = 128, N = 16 (reference; tc05_issue.cu mode 2)
//   mode 1: cta_group::2, M = 256, N = 16, leader CTA issues, commit multicast
// for 1 and 74 clusters (148 SMs).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1903_03640_b200/csrc/tcr_sm100.cuh"

using namespace tcr::sm100;

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
__device__ __forceinline__ void mma_f16_ss_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_addr(bar)), "h"((uint16_t)3)
        : "memory");
}
// bounded wait: gives up after ~2 s so a protocol mistake cannot hang the GPU
__device__ __forceinline__ bool wait_bounded(uint64_t* bar, uint32_t parity) {
    const unsigned long long t0 = now();
    while (!mbar_try_wait(bar, parity))
        if (now() - t0 > 2000000000ull) return false;
    return true;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_test(int mode, int groups, unsigned long long* out, int* err) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem);
    uint64_t* fin = cbar + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 64);
    uint8_t* a = smem + 1024;
    uint8_t* b = smem + 1024 + 65536;
    for (int i = threadIdx.x; i < (65536 + 512) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(a)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(cbar, 1);
        mbar_init(fin, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        if (mode == 1) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                             smem_addr(tslot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            tmem_alloc(tslot, 32);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // barriers initialised and TMEM allocated in both CTAs
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint64_t bdesc = smem_desc_kmajor(smem_addr(b), 128, 256);
    const uint64_t a0 = smem_desc_kmajor(smem_addr(a), 128, 256);
    bool ok = true;
    if (threadIdx.x == 0 && (mode == 0 || rank == 0)) {
        const uint32_t idesc = idesc_f16_f32(mode == 1 ? 256 : 128, 16);
        const unsigned long long t0 = now();
        for (int g = 0; g < groups; ++g) {
            for (int k = 0; k < 4; ++k) {
                const uint64_t ad = a0 + (uint64_t)(((g & 3) * 4 + k) * 256);
                if (mode == 1) mma_f16_ss_pair(tmem, ad, bdesc, idesc, 1u);
                else mma_f16_ss(tmem, ad, bdesc, idesc, 1u);
            }
            if (mode == 1) commit_pair(cbar);
            else mma_commit(cbar);
        }
        const unsigned long long t1 = now();
        if (mode == 1) commit_pair(fin);
        else mma_commit(fin);
        out[blockIdx.x] = t1 - t0;
    }
    if (threadIdx.x == 0) ok = wait_bounded(fin, 0);  // every CTA: all MMAs done
    if (!ok) atomicExch(err, 1);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) {
        if (mode == 1)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 32;" ::"r"(tmem)
                         : "memory");
        else
            tmem_dealloc(tmem, 32);
    }
}

int main() {
    unsigned long long* out;
    int* err;
    cudaMalloc(&out, 8 * 148);
    cudaMalloc(&err, 4);
    cudaMemset(err, 0, 4);
    const int smem = 1024 + 65536 + 1024;
    cudaFuncSetAttribute(pair_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int groups = 2000;
    for (int mode = 0; mode <= 1; ++mode) {
        for (int grid : {2, 148}) {
            pair_test<<<grid, 128, smem>>>(mode, groups, out, err);
            cudaError_t e = cudaDeviceSynchronize();
            int h_err = 0;
            cudaMemcpy(&h_err, err, 4, cudaMemcpyDeviceToHost);
            if (e || h_err) {
                printf("mode %d grid %d: error %s, timeout %d\n", mode, grid, cudaGetErrorString(e),
                       h_err);
                return 1;
            }
            unsigned long long h[148];
            cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
            double ns = (double)h[0] / groups;
            printf("mode %d (%s) grid %3d: %.1f ns per group of 4 MMAs (issuing thread), "
                   "%.1f GB/s of A per issuer\n",
                   mode, mode ? "cta_group::2 M=256" : "cta_group::1 M=128", grid, ns,
                   4.0 * (mode ? 8192 : 4096) / ns);
        }
    }
    return 0;
}
