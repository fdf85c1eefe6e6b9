// tc05_issue.cu -- diagnostic (not part of libtcr): cost of the MMA-issuer
// loop of the tcgen05 reduction, piece by piece, on one SM.
//   mode 0: back-to-back MMAs (groups of 4), no sync
//   mode 1: + wait on an already-complete mbarrier + fence::after_thread_sync per group
//   mode 2: + tcgen05.commit to an mbarrier per group
//   mode 3: mode 2 with 4 extra warps sleeping in mbarrier try_wait loops
//   mode 4: mode 2 with D address rotating over 16 accumulators per MMA
//   mode 5: mode 2, issue from a whole warp with elect.sync (all lanes loop)
//   mode 6: mode 2 issued concurrently by 2 warps (disjoint accumulators)
//   mode 7: mode 2 issued concurrently by 4 warps (disjoint accumulators)
// Reports issuing-thread nanoseconds per group of 4 MMAs (globaltimer).
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

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(p));
    return p != 0;
}

__global__ void __launch_bounds__(192, 1) issue_test(int mode, int groups, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* done = reinterpret_cast<uint64_t*>(smem);
    uint64_t* never = done + 1;
    uint64_t* cbar = done + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 64);
    uint8_t* a = smem + 1024;
    uint8_t* b = smem + 1024 + 65536;
    for (int i = threadIdx.x; i < (65536 + 512) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(a)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(done, 1);
        mbar_init(never, 1);
        mbar_init(cbar, 1);
        fence_mbar_init();
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 1) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) mbar_arrive(done);  // phase 0 of `done` completes
    __syncthreads();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16_f32(128, 16);
    const uint64_t bdesc = smem_desc_kmajor(smem_addr(b), 128, 256);
    const uint64_t a0 = smem_desc_kmajor(smem_addr(a), 128, 256);
    const int issuers = mode == 6 ? 2 : (mode == 7 ? 4 : 1);
    if (warp >= 1 && warp < 1 + issuers && (mode == 5 || lane == 0)) {
        unsigned long long t0 = now();
        int slot = 0;
        for (int g = 0; g < groups; ++g) {
            if (mode >= 1) {
                mbar_wait(done, 0);
                tc_fence_after();
            }
            for (int k = 0; k < 4; ++k) {
                uint32_t d = tmem + (uint32_t)(warp - 1) * 64;
                if (mode == 4) {
                    d = tmem + (uint32_t)slot * 16;
                    slot = (slot + 1) & 15;
                }
                const uint64_t ad = a0 + (uint64_t)(((g & 3) * 4 + k) * 256);
                if (mode == 5) {
                    if (elect_one()) mma_f16_ss(d, ad, bdesc, idesc, 1u);
                } else {
                    mma_f16_ss(d, ad, bdesc, idesc, 1u);
                }
            }
            if (mode >= 2) {
                if (mode != 5 || elect_one()) mma_commit(cbar + (warp - 1) * 0);
            }
        }
        unsigned long long t1 = now();
        if ((mode != 5 || lane == 0) && warp == 1) {
            out[blockIdx.x * 2] = t1 - t0;
        }
    } else if (mode == 3 && warp >= 2) {
        // sleepers: wait on a barrier that completes only when the issuer is done
        while (!mbar_try_wait(never, 0)) {
        }
    }
    __syncwarp();
    if (warp == 1 && lane == 0 && mode == 3) mbar_arrive(never);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 16 * 148);
    cudaFuncSetAttribute(issue_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 65536 + 1024);
    const int groups = 2000;
    for (int mode = 0; mode <= 7; ++mode) {
        for (int grid : {1, 148}) {
            issue_test<<<grid, 192, 1024 + 65536 + 1024>>>(mode, groups, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) {
                printf("mode %d error %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            unsigned long long h;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("mode %d grid %3d: %.1f ns per group of 4 MMAs (issuing thread)\n", mode, grid,
                   (double)h / groups);
        }
    }
    return 0;
}
