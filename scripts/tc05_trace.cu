// tc05_trace.cu -- diagnostic (not part of libtcr): timeline of CTA 0 of the
// tcgen05 reduction kernel, compiled from the library's own source with
// -DTCR_TC05_TRACE.  Usage: tc05_trace [stages] [stage_kb] [slots] [chain] [ctas] [log2 n]
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//        -DTCR_TC05_TRACE -o scripts/tc05_trace scripts/tc05_trace.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1903_03640_b200/csrc/tcr_tcgen05.cu"

int main(int argc, char** argv) {
    tcr::LaunchCfg cfg{};
    cudaDeviceGetAttribute(&cfg.sms, cudaDevAttrMultiProcessorCount, 0);
    cfg.tc05_stages = argc > 1 ? atoi(argv[1]) : 8;
    cfg.tc05_stage_kb = argc > 2 ? atoi(argv[2]) : 16;
    cfg.tc05_slots = argc > 3 ? atoi(argv[3]) : 16;
    cfg.tc05_chain = argc > 4 ? atoi(argv[4]) : 4;
    cfg.tc05_ctas = argc > 5 ? atoi(argv[5]) : 1;
    cfg.tc05_prefetch = 0;
    cfg.tc05_split = 1;
    cfg.tc05_interleave = 0;
    cfg.tc05_dynamic = getenv("TRACE_DYN") ? atoi(getenv("TRACE_DYN")) : 0;
    const size_t n = argc > 6 ? ((size_t)1 << atoi(argv[6])) : ((size_t)1 << 30);
    uint16_t* x;
    cudaMalloc(&x, n * 2);
    cudaMemset(x, 0x3C, n * 2);
    tcr::DevWorkspace ws{};
    cudaMalloc(&ws.partials, 8 * 4096);
    cudaMalloc(&ws.ticket, 64);
    cudaMemset(ws.ticket, 0, 64);
    cudaMalloc(&ws.chunk_next, 64);
    cudaMemset(ws.chunk_next, 0, 64);
    ws.capacity = 4096;
    float* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int r = 0, R_ = getenv("TRACE_REPS") ? atoi(getenv("TRACE_REPS")) : 5; r < R_; ++r) {
        cudaEventRecord(a);
        cudaError_t e = tcr::launch_reduce_tcgen05(getenv("TRACE_FMT") ? atoi(getenv("TRACE_FMT")) : 0, x, n, out, nullptr, ws, cfg, 0);
        cudaEventRecord(b);
        if (e || (e = cudaDeviceSynchronize())) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaEventElapsedTime(&ms, a, b);
    }
    printf("cfg stages=%d kb=%d slots=%d chain=%d ctas=%d dyn=%d: %.1f us, %.1f GB/s\n", cfg.tc05_stages,
           cfg.tc05_stage_kb, cfg.tc05_slots, cfg.tc05_chain, cfg.tc05_ctas, cfg.tc05_dynamic, ms * 1e3,
           n * 2 / (ms * 1e-3) / 1e9);
    static unsigned long long tr[6][4096];
    cudaMemcpyFromSymbol(tr, tcr::g_tc05_trace, sizeof(tr));
    const int nch = (int)((n * 2 / (cfg.tc05_stage_kb * 1024)) / (cfg.sms * cfg.tc05_ctas));
    const int m = std::min(nch, 4096);
    const unsigned long long t0 = tr[0][0];
    auto pct = [](std::vector<double> v, double p) {
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[(size_t)(p * (v.size() - 1))];
    };
    std::vector<double> issue_gap, tma_lat, mma_time, full_gap;
    for (int i = 1; i < m; ++i) {
        issue_gap.push_back((double)(tr[0][i] - tr[0][i - 1]));
        full_gap.push_back((double)(tr[1][i] - tr[1][i - 1]));
    }
    for (int i = 0; i < m; ++i) {
        tma_lat.push_back((double)(tr[1][i] - tr[0][i]));
        mma_time.push_back((double)(tr[2][i] - tr[1][i]));
    }
    printf("chunks/CTA %d; ns: producer issue gap p50 %.0f p90 %.0f | issue->full p50 %.0f p90 %.0f | "
           "full->committed p50 %.0f p90 %.0f | full gap p50 %.0f p90 %.0f\n",
           nch, pct(issue_gap, .5), pct(issue_gap, .9), pct(tma_lat, .5), pct(tma_lat, .9),
           pct(mma_time, .5), pct(mma_time, .9), pct(full_gap, .5), pct(full_gap, .9));
    printf("first 24 chunks (ns from first issue): i issue full committed\n");
    for (int i = 0; i < std::min(m, 24); ++i)
        printf("  %3d %8llu %8llu %8llu\n", i, tr[0][i] - t0, tr[1][i] - t0, tr[2][i] - t0);
    printf("epilogue rounds (ns): ");
    for (int r = 0; r < 12; ++r) printf("%llu ", tr[3][r] - t0);
    printf("\nlast chunk committed at %llu ns\n", tr[2][m - 1] - t0);
    printf("MMA issue times (ns from first issue), first 40: ");
    for (int i = 0; i < 40; ++i) printf("%llu ", tr[4][i] - t0);
    printf("\ntempty seen per round, first 12: ");
    for (int r = 0; r < 12; ++r) printf("%llu ", tr[5][r] - t0);
    std::vector<double> mg;
    for (int i = 1; i < 4000; ++i) mg.push_back((double)(tr[4][i] - tr[4][i - 1]));
    printf("\nMMA issue gap p10 %.0f p50 %.0f p90 %.0f ns\n", pct(mg, .1), pct(mg, .5), pct(mg, .9));
    // per-CTA phase edges of the last launch, relative to the earliest entry
    static unsigned long long ed[10][2048];
    cudaMemcpyFromSymbol(ed, tcr::g_tc05_edges, sizeof(ed));
    const int G = std::min(tcr::tcgen05_grid(n * 2, cfg), 2048);
    unsigned long long e0 = ~0ull, eend = 0;
    for (int b = 0; b < G; ++b) {
        e0 = std::min(e0, ed[0][b]);
        eend = std::max(eend, ed[3][b]);
    }
    std::vector<double> ent, setup, data, fin;
    for (int b = 0; b < G; ++b) {
        ent.push_back((double)(ed[0][b] - e0));
        setup.push_back((double)(ed[1][b] - ed[0][b]));
        data.push_back((double)(ed[2][b] - e0));
        fin.push_back((double)(ed[3][b] - ed[2][b]));
    }
    printf("CTAs %d: entry p0 %.0f p50 %.0f p100 %.0f | setup p50 %.0f p100 %.0f | data done p0 %.0f "
           "p50 %.0f p100 %.0f | completion p50 %.0f p100 %.0f | last exit %.0f ns\n",
           G, pct(ent, 0), pct(ent, 0.5), pct(ent, 1), pct(setup, 0.5), pct(setup, 1), pct(data, 0),
           pct(data, 0.5), pct(data, 1), pct(fin, 0.5), pct(fin, 1), (double)(eend - e0));
    printf("data done deciles (ns):");
    for (int q = 0; q <= 10; ++q) printf(" %.0f", pct(data, q / 10.0));
    printf("\n");
    {  // dynamic-tail completion: 8 = ticket returned (thread 0), 9 = after the CTA barrier
        std::vector<double> d89;
        for (int b = 0; b < G; ++b) d89.push_back((double)(ed[9][b] - ed[8][b]));
        printf("dyn completion barrier after the ticket: 8->9 p50 %.0f p100 %.0f ns\n", pct(d89, .5),
               pct(d89, 1));
    }
    // completion steps: 2 data done -> 4 warp collapse -> 5 syncthreads -> 6 CTA collapse
    // -> 7 partial stored + threadfence -> 8 ticket returned -> 3 exit
    const int ks[7] = {2, 4, 5, 6, 7, 8, 3};
    printf("completion step p50 / p100 (ns):");
    for (int i = 0; i + 1 < 7; ++i) {
        std::vector<double> d;
        for (int b = 0; b < G; ++b) d.push_back((double)(ed[ks[i + 1]][b] - ed[ks[i]][b]));
        printf("  %d->%d %.0f/%.0f", ks[i], ks[i + 1], pct(d, 0.5), pct(d, 1));
    }
    printf("\n");
    return 0;
}
