// tc05_borient.cu -- diagnostic (not part of libtcr): per-instruction cost of
// tcgen05.mma for the two orientations of the level-1 reduction on B200
// ("changing the order of the multiplying
// matrices"):
//   A-orient: A = input tile (128 x 16, 4 KiB), B = ones (N x 16), D = 128 x N
//             (row sums, replicated over N columns)   -- the r01 kernel, N = 16
//   B-orient: A = ones (128 x 16), B = input (N x 16 = N*32 bytes), D = 128 x N
//             (column sums, replicated over 128 rows) -- input bytes per MMA
//             grow with N (8 KiB at N = 256)
// One issuing thread per SM, groups of 4 MMAs + tcgen05.commit per group (as
// the pipeline does), 1 CTA per SM on all SMs.  Prints ns per MMA (globaltimer,
// issuing thread, max over SMs) and input GB/s per SM and per chip.  Also
// checks the B-orient numerics once: D[0][n] == sum_k B[n][k].
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1903_03640_b200/csrc/tcr_sm100.cuh"

using namespace tcr::sm100;

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(p));
    return p != 0;
}

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// bounded wait: gives up after 20 ms (a diagnostic must never hang the GPU)
__device__ bool g_timed_out = false;
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
    const unsigned long long t0 = now();
    while (!mbar_try_wait(bar, parity)) {
        if (now() - t0 > 20000000ull) { g_timed_out = true; return; }
    }
}

// smem: [0,1024) barriers; [1024, +64K) input tiles; [+64K, +8K) ones
__global__ void __launch_bounds__(128, 1) rate(int borient, int N, int groups, unsigned long long* out,
                                               float* dcheck, int inflight, int slots, int warpissue) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem);  // [inflight <= 8]: one per group slot
    uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + 64);
    uint8_t* in = smem + 1024;
    uint8_t* ones = smem + 1024 + 65536;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(in)[i] = 0x3C003C00u;
    for (int i = threadIdx.x; i < 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(ones)[i] = 0x3C003C00u;
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int b = 0; b < inflight; ++b) mbar_init(&cbar[b], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc(tslot, 512);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t idesc = idesc_f16_f32(128, N);
    const uint32_t in_bytes = borient ? (uint32_t)N * 32 : 4096u;  // input bytes per MMA
    const int tiles = 65536 / (int)in_bytes;
    // warpissue: the whole warp 0 runs the issue loop (warp-uniform values ->
    // uniform registers) and elect.sync picks the issuing lane per MMA;
    // otherwise thread 0 alone (ptxas then wraps every tcgen05.mma in an
    // R2UR + elect waterfall)
    const int warp_u = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0);  // provably warp-uniform
    if (warpissue ? warp_u == 0 : threadIdx.x == 0) {
        const uint64_t onesd = smem_desc_kmajor(smem_addr(ones), 128, 256);
        const uint64_t in0 = smem_desc_kmajor(smem_addr(in), 128, 256);
        // group g commits to cbar[g % inflight]; before reusing a barrier,
        // wait for its previous phase (group g - inflight), so no barrier ever
        // runs more than one phase ahead of its waiter
        uint32_t ph[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        const unsigned long long t0 = now();
        for (int g = 0; g < groups; ++g) {
            const int b = g % inflight;
            if (g >= inflight) { mbar_wait_bounded(&cbar[b], ph[b]); ph[b] ^= 1u; }
            for (int k = 0; k < 4; ++k) {
                const int j = g * 4 + k;
                const uint64_t idd = in0 + (uint64_t)(((j & (tiles - 1)) * in_bytes) >> 4);  // powers of two: no integer division in the issue loop
                const uint32_t d = tmem + (uint32_t)((j & (slots - 1)) * N);
                const uint32_t acc = j >= slots ? 1u : 0u;
                if (warpissue) {
                    if (elect_one()) {
                        if (borient) mma_f16_ss(d, onesd, idd, idesc, acc);
                        else mma_f16_ss(d, idd, onesd, idesc, acc);
                    }
                    __syncwarp();
                } else if (borient) {
                    mma_f16_ss(d, onesd, idd, idesc, acc);
                } else {
                    mma_f16_ss(d, idd, onesd, idesc, acc);
                }
            }
            if (!warpissue) {
                mma_commit(&cbar[b]);
            } else {
                if (elect_one()) mma_commit(&cbar[b]);
                __syncwarp();  // whole warp 0 only (never from the lone thread-0 issuer)
            }
        }
        for (int g = groups > inflight ? groups - inflight : 0; g < groups; ++g) {
            const int b = g % inflight;
            mbar_wait_bounded(&cbar[b], ph[b]);
            ph[b] ^= 1u;
        }
        const unsigned long long t1 = now();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (blockIdx.x == 0 && threadIdx.x < 32 && dcheck) {
        // lane t: D[t][0..16) of accumulator 0 (every entry should be 16 * (#MMAs into slot 0))
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tmem));
        tmem_wait_ld();
        for (int c = 0; c < 16; ++c) dcheck[threadIdx.x * 16 + c] = __uint_as_float(v[c]);
    }
    tc_fence_before(); __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out; cudaMalloc(&out, 8 * sms);
    float* dc; cudaMalloc(&dc, 4 * 512);
    const size_t smem = 1024 + 65536 + 8192;
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int groups = 4000;
    for (int wi = 0; wi < 2; ++wi) {
    for (int bo = 0; bo < 2; ++bo) {
        for (int N : {16, 64, 256}) {
            for (int inflight : {2, 4}) {
                for (int slots : {2, 4}) {
                    if (slots * N > 512) continue;
                    rate<<<sms, 128, smem>>>(bo, N, groups, out, (bo && slots == 2) ? dc : nullptr,
                                             inflight, slots, wi);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                    unsigned long long h[256]; cudaMemcpy(h, out, 8 * sms, cudaMemcpyDeviceToHost);
                    unsigned long long mx = 0; for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
                    const double ns = (double)mx / (4.0 * groups);
                    const double bytes = bo ? N * 32.0 : 4096.0;
                    printf("%s %s N=%3d inflight=%d slots=%2d: %6.1f ns/MMA  %5.0f B/MMA  %6.1f GB/s/SM  %6.0f GB/s chip",
                           wi ? "warp+elect " : "thread0    ", bo ? "B-orient (ones x X)" : "A-orient (X x ones)", N,
                           inflight, slots, ns, bytes, bytes / ns, bytes / ns * sms);
                    if (bo && slots == 2) {
                        float hd[512]; cudaMemcpy(hd, dc, 4 * 512, cudaMemcpyDeviceToHost);
                        printf("  D[0][0]=%g D[31][15]=%g (expect %d)", hd[0], hd[31 * 16 + 15], 16 * 2 * groups);
                    }
                    bool to = false;
                    cudaMemcpyFromSymbol(&to, g_timed_out, sizeof(bool));
                    printf("%s\n", to ? "  TIMED OUT (bounded wait)" : "");
                    fflush(stdout);
                    if (to) return 3;
                }
            }
        }
    }
    }
    return 0;
}
