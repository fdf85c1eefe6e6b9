// stream_trace.cu -- diagnostic (not part of libtcr): per-CTA phase edges of
// the default mma.sync streaming kernel, compiled from the library's source
// with TCR_COMPLETE_EDGE recording %globaltimer.  Usage: stream_trace [log2 n] [bps]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace tcr {
__device__ unsigned long long g_edges[10][4096];
}
#define TCR_COMPLETE_EDGE(k)                                                        \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 4096) {                                \
            unsigned long long t_;                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
            tcr::g_edges[k][blockIdx.x] = t_;                                       \
        }                                                                           \
    } while (0)
#include "../paper_1903_03640_b200/csrc/tcr_reduce.cu"

int main(int argc, char** argv) {
    tcr::LaunchCfg cfg{};
    cudaDeviceGetAttribute(&cfg.sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n = (size_t)1 << (argc > 1 ? atoi(argv[1]) : 30);
    cfg.blocks_per_sm = argc > 2 ? atoi(argv[2]) : 8;
    cfg.unroll = 0;
    cfg.chain = 4;
    uint16_t* x;
    cudaMalloc(&x, n * 2);
    cudaMemset(x, 0x3C, n * 2);
    tcr::DevWorkspace ws{};
    cudaMalloc(&ws.partials, 8 * 8192);
    cudaMalloc(&ws.ticket, 64);
    cudaMemset(ws.ticket, 0, 64);
    ws.capacity = 8192;
    float* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int r = 0, R_ = getenv("TRACE_REPS") ? atoi(getenv("TRACE_REPS")) : 5; r < R_; ++r) {
        cudaEventRecord(a);
        cudaError_t e = tcr::launch_reduce_stream(true, 0, x, n, out, nullptr, ws, cfg, 0);
        cudaEventRecord(b);
        if (e || (e = cudaDeviceSynchronize())) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaEventElapsedTime(&ms, a, b);
    }
    static unsigned long long ed[10][4096];
    cudaMemcpyFromSymbol(ed, tcr::g_edges, sizeof(ed));
    tcr::LaunchCfg c2 = cfg;
    c2.unroll = n < ((size_t)1 << 26) ? 16 : 4;
    const int G = std::min(tcr::stream_grid(n, c2), 4096);
    auto pct = [](std::vector<double> v, double p) {
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[(size_t)(p * (v.size() - 1))];
    };
    unsigned long long e0 = ~0ull, eend = 0;
    for (int i = 0; i < G; ++i) {
        e0 = std::min(e0, ed[0][i]);
        eend = std::max(eend, ed[3][i]);
    }
    std::vector<double> ent, done, fin;
    for (int i = 0; i < G; ++i) {
        ent.push_back((double)(ed[0][i] - e0));
        done.push_back((double)(ed[2][i] - e0));
        fin.push_back((double)(ed[3][i] - ed[2][i]));
    }
    printf("n=2^%d grid %d: %.1f us (events) | entry p50 %.0f p100 %.0f | data done p0 %.0f p50 %.0f "
           "p100 %.0f | completion p50 %.0f p100 %.0f | last exit %.0f ns\n",
           (int)(63 - __builtin_clzll(n)), G, ms * 1e3, pct(ent, .5), pct(ent, 1), pct(done, 0),
           pct(done, .5), pct(done, 1), pct(fin, .5), pct(fin, 1), (double)(eend - e0));
    printf("  data done deciles (ns):");
    for (int q = 0; q <= 10; ++q) printf(" %.0f", pct(done, q / 10.0));
    printf("\n");
    const int ks[7] = {2, 4, 5, 6, 7, 8, 3};
    printf("  completion step p50 / p100 (ns):");
    for (int i = 0; i + 1 < 7; ++i) {
        std::vector<double> d;
        for (int b2 = 0; b2 < G; ++b2)
            if (ed[ks[i + 1]][b2] >= ed[ks[i]][b2]) d.push_back((double)(ed[ks[i + 1]][b2] - ed[ks[i]][b2]));
        printf("  %d->%d %.0f/%.0f", ks[i], ks[i + 1], pct(d, .5), pct(d, 1));
    }
    printf("\n");
    return 0;
}
