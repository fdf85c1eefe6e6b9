// dmma_latency.cu -- diagnostic (not part of libtcr): latency of the level-2
// collapse D' = 1 x D (three m8n8k4 f64 DMMAs, warp_collapse_mma) vs the
// shfl_xor tree, measured by one warp per SM with %globaltimer:
//   at kernel start (cold), after a ~busy-wait (idle FP64 pipe), and back to back.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_1903_03640_b200/csrc/tcr_device.cuh"

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void lat_kernel(int mode, long long spin_ns, unsigned long long* out, double* sink) {
    const int lane = threadIdx.x & 31;
    double v = (double)lane + 0.5;
    if (spin_ns) {  // idle the FP64 pipe for spin_ns
        const unsigned long long t0 = now();
        while (now() - t0 < (unsigned long long)spin_ns) {
        }
    }
    __syncwarp();
    unsigned long long t0 = now();
    double r = 0.0;
    for (int rep = 0; rep < 3; ++rep) {
        r = mode == 0 ? tcr::warp_collapse_mma(v + r) : tcr::warp_collapse_shfl(v + r);
    }
    __syncwarp();
    unsigned long long t1 = now();
    if (lane == 0) {
        out[blockIdx.x] = t1 - t0;
        sink[blockIdx.x] = r;
    }
}

int main() {
    unsigned long long* out;
    double* sink;
    cudaMalloc(&out, 8 * 148);
    cudaMalloc(&sink, 8 * 148);
    for (int mode = 0; mode < 2; ++mode)
        for (long long spin : {0LL, 1000LL, 10000LL, 100000LL, 1000000LL}) {
            for (int rep = 0; rep < 3; ++rep) {
                lat_kernel<<<148, 32>>>(mode, spin, out, sink);
                cudaDeviceSynchronize();
            }
            unsigned long long h[148];
            cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0, sum = 0;
            for (int i = 0; i < 148; ++i) {
                sum += h[i];
                if (h[i] > mx) mx = h[i];
            }
            printf("%s after %7lld ns idle: 3 collapses mean %6.0f ns, max %6llu ns\n",
                   mode == 0 ? "DMMA collapse" : "shfl collapse", spin, sum / 148.0, mx);
        }
    return 0;
}
