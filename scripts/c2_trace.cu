// c2_trace.cu -- diagnostic (not part of libtcr): where the time of one
// BASELINE config 2 launch (n = 2^24 fp16, 32 MiB) goes, cold and warm.
// The library's streaming kernel is compiled from its source with
// TCR_COMPLETE_EDGE recording %globaltimer per CTA (thread 0).
//
// Timing discipline: every timed launch is queued behind a ~40 us spin
// kernel, so the host's launch cost is hidden and the event pair measures
// the GPU side only (front-end launch + kernel).  Modes:
//   warm       -- x resident in L2 (previous launch read it)
//   cold_clean -- a 512 MiB read-only sweep between launches (x evicted, L2
//                 full of clean lines)
//   empty      -- an empty kernel of the same grid (the launch floor)
//   b2b        -- 200 back-to-back launches between one event pair (warm),
//                 per-launch average: what a caller issuing calls in a row sees
// usage: c2_trace [log2 n] [reps] [pdl 0/1 (trees with TCR_CFG_PDL)]
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
// built twice by scripts/runs/r2_c2ab.sh: -I <a csrc tree> selects the kernel source
#include "tcr_reduce.cu"

__global__ void spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while ((long long)(t - t0) < ns);
}
__global__ void empty_k() {}
__global__ void sweep(const uint4* p, size_t nv, unsigned* sink) {
    unsigned a = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcg(p + i);
        a ^= v.x ^ v.w;
    }
    if (a == 0x7355608u) *sink = a;
}

int main(int argc, char** argv) {
    tcr::LaunchCfg cfg{};
    cudaDeviceGetAttribute(&cfg.sms, cudaDevAttrMultiProcessorCount, 0);
    const int lg = argc > 1 ? atoi(argv[1]) : 24;
    const int reps = argc > 2 ? atoi(argv[2]) : 50;
    const size_t n = (size_t)1 << lg;
    cfg.blocks_per_sm = 8;
    cfg.unroll = 0;
    cfg.chain = 4;
#ifdef TCR_HAS_PDL
    cfg.pdl = argc > 3 ? atoi(argv[3]) : 1;
#endif
    uint16_t* x;
    cudaMalloc(&x, n * 2);
    cudaMemset(x, 0x3C, n * 2);
    const size_t fb = (size_t)512 << 20;
    uint4* fl;
    unsigned* sink;
    cudaMalloc(&fl, fb);
    cudaMemset(fl, 1, fb);
    cudaMalloc(&sink, 4);
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
    tcr::LaunchCfg c2 = cfg;
    c2.unroll = n < ((size_t)1 << 26) ? 16 : 4;
    const int G = std::min(tcr::stream_grid(n, c2), 4096);
    auto pct = [](std::vector<double> v, double p) {
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[(size_t)(p * (v.size() - 1))];
    };
    {
        for (int r = 0; r < 20; ++r) tcr::launch_reduce_stream(true, 0, x, n, out, nullptr, ws, cfg, 0);
        cudaEventRecord(a);
        for (int r = 0; r < 200; ++r) tcr::launch_reduce_stream(true, 0, x, n, out, nullptr, ws, cfg, 0);
        cudaEventRecord(b);
        cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("n=2^%d grid %d b2b        %.2f us per launch (200 back-to-back, warm)\n", lg, G,
               ms * 1e3 / 200);
    }
    for (int mode = 0; mode < 3; ++mode) {
        const char* name = mode == 0 ? "warm" : mode == 1 ? "cold_clean" : "empty";
        std::vector<double> ev, body, ent, dn, dn100, ex_after_data, first_data;
        std::vector<std::vector<double>> steps(6);
        const int ks[7] = {2, 4, 5, 6, 7, 8, 3};
        for (int r = 0; r < reps + 3; ++r) {
            if (mode == 1) sweep<<<cfg.sms * 8, 256>>>(fl, fb / 16, sink);
            else if (mode == 0) tcr::launch_reduce_stream(true, 0, x, n, out, nullptr, ws, cfg, 0);
            spin<<<1, 32>>>(40000);
            cudaEventRecord(a);
            if (mode == 2) empty_k<<<G, 256>>>();
            else tcr::launch_reduce_stream(true, 0, x, n, out, nullptr, ws, cfg, 0);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            if (r < 3) continue;
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            ev.push_back(ms * 1e3);
            if (mode == 2) continue;
            static unsigned long long ed[10][4096];
            cudaMemcpyFromSymbol(ed, tcr::g_edges, sizeof(ed));
            unsigned long long e0 = ~0ull, eend = 0, dmax = 0;
            for (int i = 0; i < G; ++i) {
                e0 = std::min(e0, ed[0][i]);
                eend = std::max(eend, ed[3][i]);
                dmax = std::max(dmax, ed[2][i]);
            }
            body.push_back((eend - e0) / 1e3);
            std::vector<double> en, d;
            for (int i = 0; i < G; ++i) {
                en.push_back((double)(ed[0][i] - e0));
                d.push_back((double)(ed[2][i] - e0));
            }
            ent.push_back(pct(en, 1.0) / 1e3);
            dn.push_back(pct(d, 0.5) / 1e3);
            dn100.push_back(pct(d, 1.0) / 1e3);
            first_data.push_back(pct(d, 0.0) / 1e3);
            ex_after_data.push_back((eend - dmax) / 1e3);
            for (int s = 0; s < 6; ++s) {
                std::vector<double> st;
                for (int i = 0; i < G; ++i)
                    if (ed[ks[s + 1]][i] >= ed[ks[s]][i]) st.push_back((double)(ed[ks[s + 1]][i] - ed[ks[s]][i]));
                steps[s].push_back(pct(st, 1.0));
            }
        }
        auto med = [&](std::vector<double> v) { return pct(v, 0.5); };
        printf("n=2^%d grid %d %-10s events %.2f us", lg, G, name, med(ev));
        if (mode != 2) {
            printf(" | kernel body (first entry..last exit) %.2f | last CTA entry %.2f | data done "
                   "p0 %.2f p50 %.2f p100 %.2f | last exit after last data %.2f us\n",
                   med(body), med(ent), med(first_data), med(dn), med(dn100), med(ex_after_data));
            printf("    completion steps p100 (ns, median over reps):");
            for (int s = 0; s < 6; ++s) printf("  %d->%d %.0f", ks[s], ks[s + 1], med(steps[s]));
            printf("\n");
        } else {
            printf("  (launch floor: empty kernel of the same grid)\n");
        }
    }
    return 0;
}
