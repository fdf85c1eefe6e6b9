/*
 * c_api_demo.c -- using libtcr from plain C (no Python, no torch): allocate
 * device memory with the CUDA runtime, fill it, and call the C ABI of
 * include/tcr.h.  Prints the MMA-encoded, shuffle, exact and (one-rank)
 * peer-combined sums of
 * x_i = ((i % 7) - 3) * 0.25 for i < n (exactly representable; the exact sum
 * is known in closed form, so the program checks itself).
 *
 * Build: gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *        -L paper_1903_03640_b200 -ltcr -L /usr/local/cuda/lib64 -lcudart \
 *        -Wl,-rpath,$PWD/paper_1903_03640_b200 -o examples/c_api_demo
 * Usage: examples/c_api_demo [n]
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tcr.h"

static uint16_t quarter_bits(int q) { /* binary16 of q * 0.25 for q in [-3, 3] */
    static const uint16_t tab[7] = {0xBA00, 0xB800, 0xB400, 0x0000, 0x3400, 0x3800, 0x3A00};
    return tab[q + 3];
}

#define CHECK(call)                                                                     \
    do {                                                                                \
        tcr_status s_ = (call);                                                         \
        if (s_ != TCR_OK) {                                                             \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, tcr_status_string(s_),       \
                    tcr_last_error());                                                  \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? (size_t)strtoull(argv[1], 0, 10) : ((size_t)1 << 24) + 3;
    uint16_t* h = (uint16_t*)malloc(n * sizeof(uint16_t));
    long long exact_q = 0; /* sum in units of 0.25 */
    for (size_t i = 0; i < n; ++i) {
        const int q = (int)(i % 7) - 3;
        h[i] = quarter_bits(q);
        exact_q += q;
    }
    tcr_half* x = 0;
    float* out = 0;
    int64_t* acc = 0;
    if (cudaMalloc((void**)&x, n * sizeof(uint16_t)) || cudaMalloc((void**)&out, 4 * sizeof(float)) ||
        cudaMalloc((void**)&acc, 6 * sizeof(int64_t))) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(x, h, n * sizeof(uint16_t), cudaMemcpyHostToDevice);
    CHECK(tcr_reduce_sum(x, n, out, 0));
    CHECK(tcr_reduce_sum_shuffle(x, n, out + 1, 0));
    CHECK(tcr_reduce_sum_exact(x, n, acc, out + 2, 0, 0));
    /* a one-rank peer group: the fused cross-GPU combine with itself */
    void* mailbox = 0;
    CHECK(tcr_peer_mailbox_alloc(&mailbox));
    CHECK(tcr_reduce_sum_peer(x, n, TCR_DTYPE_F16, TCR_ALGO_DEFAULT, &mailbox, 1, 0, out + 3, 0, 0));
    float r[4];
    cudaMemcpy(r, out, sizeof r, cudaMemcpyDeviceToHost);
    float host_r = 0;
    CHECK(tcr_reduce_sum_host(h, n, &host_r, 0));
    const double want = 0.25 * (double)exact_q;
    printf("n=%zu exact=%.2f mma=%.2f shuffle=%.2f exact_gpu=%.2f peer=%.2f host_entry=%.2f "
           "launches=%llu\n",
           n, want, r[0], r[1], r[2], r[3], host_r, (unsigned long long)tcr_launch_count());
    const int ok = r[0] == (float)want && r[1] == (float)want && r[2] == (float)want &&
                   r[3] == (float)want && host_r == (float)want;
    tcr_peer_mailbox_free(mailbox);
    tcr_release_workspaces();
    cudaFree(x);
    cudaFree(out);
    cudaFree(acc);
    free(h);
    printf(ok ? "OK\n" : "MISMATCH\n");
    return ok ? 0 : 2;
}
