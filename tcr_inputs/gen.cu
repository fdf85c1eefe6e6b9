// gen.cu -- device implementation of the seeded input generator
// (tcr_inputs/__init__.py holds the host implementation and the definition).
// Holds none of the reduction's arithmetic.  Built into libtcr_inputs.so.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t pm1_bits(uint64_t seed, uint64_t i) {
    const uint64_t z = splitmix64(seed, i);
    const float v = (float)(uint32_t)(z >> 40) * 0x1p-23f - 1.0f;  // exact in binary32
    return __half_as_ushort(__float2half_rn(v));
}

__device__ __forceinline__ uint16_t gen_one(uint64_t seed, uint64_t i, int dist) {
    switch (dist) {
        case 0: return pm1_bits(seed, i);
        case 1: {
            const uint64_t z = splitmix64(seed, i);
            return __half_as_ushort(__float2half_rn((float)(uint32_t)(z >> 40) * 0x1p-24f));
        }
        case 2: return 0x3C00;
        case 3: {
            const uint16_t b = pm1_bits(seed, i & ~1ull);
            return (i & 1ull) ? (uint16_t)(b ^ 0x8000u) : b;
        }
        case 4: {
            const uint64_t z = splitmix64(seed, i);
            const uint16_t sign = (uint16_t)(z >> 63);
            const uint16_t e = (uint16_t)((z >> 32) % 31ull);
            const uint16_t f = (uint16_t)(z & 0x3FFull);
            return (uint16_t)((sign << 15) | (e << 10) | f);
        }
        default: {  // 5: small integers in {-2..2}
            const uint64_t z = splitmix64(seed, i);
            const int v = (int)((z >> 32) % 5ull) - 2;
            return __half_as_ushort(__float2half_rn((float)v));
        }
    }
}

__device__ __forceinline__ uint16_t gen_one_bf16(uint64_t seed, uint64_t i, int dist) {
    switch (dist) {
        case 0:
        case 1:
        case 3: {
            const uint64_t z = splitmix64(seed, dist == 3 ? (i & ~1ull) : i);
            const float r = (float)(uint32_t)(z >> 40);
            const float v = dist == 1 ? r * 0x1p-24f : r * 0x1p-23f - 1.0f;
            const uint16_t b = __bfloat16_as_ushort(__float2bfloat16_rn(v));
            return (dist == 3 && (i & 1ull)) ? (uint16_t)(b ^ 0x8000u) : b;
        }
        case 2: return 0x3F80;
        case 4: {
            const uint64_t z = splitmix64(seed, i);
            const uint16_t sign = (uint16_t)(z >> 63);
            const uint16_t e = (uint16_t)(64ull + (z >> 32) % 127ull);
            const uint16_t f = (uint16_t)(z & 0x7Full);
            return (uint16_t)((sign << 15) | (e << 7) | f);
        }
        default: {
            const uint64_t z = splitmix64(seed, i);
            const float v = (float)(int)((z >> 32) % 5ull) - 2.0f;
            return __bfloat16_as_ushort(__float2bfloat16_rn(v));
        }
    }
}

__global__ void gen_kernel_bf16(uint16_t* __restrict__ out, uint64_t seed, uint64_t start,
                                uint64_t count, int dist) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
        out[k] = gen_one_bf16(seed, start + k, dist);
}

__device__ __forceinline__ uint8_t gen_one_fp8(uint64_t seed, uint64_t i, int dist, int fmt) {
    const __nv_fp8_interpretation_t it = fmt == 0 ? __NV_E4M3 : __NV_E5M2;
    const int mb = fmt == 0 ? 3 : 2;
    switch (dist) {
        case 0:
        case 1:
        case 3: {
            const uint64_t z = splitmix64(seed, dist == 3 ? (i & ~1ull) : i);
            const float r = (float)(uint32_t)(z >> 40);
            const float v = dist == 1 ? r * 0x1p-24f : r * 0x1p-23f - 1.0f;
            const uint8_t b = (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, it);
            return (dist == 3 && (i & 1ull)) ? (uint8_t)(b ^ 0x80u) : b;
        }
        case 2: return fmt == 0 ? 0x38 : 0x3C;
        case 4: {
            const uint64_t z = splitmix64(seed, i);
            const int eb = 7 - mb;
            const uint8_t sign = (uint8_t)(z >> 63);
            const uint8_t e = (uint8_t)((z >> 32) % (uint64_t)((1 << eb) - 1));
            const uint8_t f = (uint8_t)(z & (uint64_t)((1 << mb) - 1));
            return (uint8_t)((sign << 7) | (e << mb) | f);
        }
        default: {
            const uint64_t z = splitmix64(seed, i);
            const float v = (float)(int)((z >> 32) % 5ull) - 2.0f;
            return (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, it);
        }
    }
}

__global__ void gen_kernel_fp8(uint8_t* __restrict__ out, uint64_t seed, uint64_t start,
                               uint64_t count, int dist, int fmt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
        out[k] = gen_one_fp8(seed, start + k, dist, fmt);
}

__global__ void gen_kernel(uint16_t* __restrict__ out, uint64_t seed, uint64_t start,
                           uint64_t count, int dist) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
        out[k] = gen_one(seed, start + k, dist);
}

}  // namespace

static int launch_gen(bool bf16, void* out, uint64_t seed, uint64_t start, uint64_t count,
                      int dist, void* stream) {
    if (count == 0) return 0;
    if (!out || dist < 0 || dist > 5) return 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (count + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    if (bf16)
        gen_kernel_bf16<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((uint16_t*)out, seed,
                                                                             start, count, dist);
    else
        gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((uint16_t*)out, seed,
                                                                        start, count, dist);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int tcr_inputs_generate(void* out, uint64_t seed, uint64_t start, uint64_t count,
                                   int dist, void* stream) {
    return launch_gen(false, out, seed, start, count, dist, stream);
}

extern "C" int tcr_inputs_generate_fp8(void* out, uint64_t seed, uint64_t start, uint64_t count,
                                       int dist, int fmt, void* stream) {
    if (count == 0) return 0;
    if (!out || dist < 0 || dist > 5 || fmt < 0 || fmt > 1) return 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t blocks = (count + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (blocks > cap) blocks = cap;
    gen_kernel_fp8<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((uint8_t*)out, seed, start,
                                                                        count, dist, fmt);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int tcr_inputs_generate_bf16(void* out, uint64_t seed, uint64_t start, uint64_t count,
                                        int dist, void* stream) {
    return launch_gen(true, out, seed, start, count, dist, stream);
}
