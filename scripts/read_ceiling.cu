// read_ceiling.cu -- diagnostic (not part of libtcr): how fast can a kernel
// READ HBM on this B200?  XOR-reduces a 2 GiB buffer with 16-byte loads at
// several unroll / occupancy settings and prints GB/s (CUDA events, best of
// 20).  Gives the "100 %" a read-only streaming reduction can reach, next to
// MEASURED_PEAKS.json's copy bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256, 4) xor_kernel(const uint4* __restrict__ p, size_t nvec, unsigned* out) {
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    size_t i = tid;
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * stride));
        __syncwarp();
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < nvec; i += stride) { uint4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    if (acc == 0x12345678u) *out = acc;
}

template <int U>
float run(const uint4* p, size_t nvec, unsigned* out, int bps, int sms) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 23; ++r) {
        cudaEventRecord(a);
        xor_kernel<U><<<sms * bps, 256>>>(p, nvec, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (r >= 3 && ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = (size_t)2 << 30;
    void* p; unsigned* out;
    cudaMalloc(&p, bytes); cudaMalloc(&out, 4);
    cudaMemset(p, 1, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t nvec = bytes / 16;
    for (int bps : {2, 4, 8}) {
        printf("bps=%d U=4  %.1f GB/s\n", bps, bytes / (run<4>((uint4*)p, nvec, out, bps, sms) * 1e-3) / 1e9);
        printf("bps=%d U=8  %.1f GB/s\n", bps, bytes / (run<8>((uint4*)p, nvec, out, bps, sms) * 1e-3) / 1e9);
        printf("bps=%d U=16 %.1f GB/s\n", bps, bytes / (run<16>((uint4*)p, nvec, out, bps, sms) * 1e-3) / 1e9);
    }
    // cudaMemcpy D2D (read + write) for reference
    void* q; cudaMalloc(&q, bytes / 2);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 13; ++r) {
        cudaEventRecord(a); cudaMemcpy(q, p, bytes / 2, cudaMemcpyDeviceToDevice); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 3 && ms < best) best = ms;
    }
    printf("memcpy D2D 1 GiB: %.1f GB/s (read+write)\n", bytes / (best * 1e-3) / 1e9);
    return 0;
}
