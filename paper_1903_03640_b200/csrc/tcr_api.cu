// tcr_api.cu -- the C ABI of libtcr (include/tcr.h): argument validation,
// device check, per-(device, stream) workspace cache, kernel dispatch.
// Every compute step runs in this library's kernels; there is no fallback.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/tcr.h"
#include "tcr_internal.h"

namespace tcr {
cudaError_t launch_probe_mma_sync(const uint16_t* a, const float* c, float* d,
                                  cudaStream_t stream);
cudaError_t launch_probe_mma_tcgen05(const uint16_t* a, const float* c, float* d,
                                     cudaStream_t stream);
cudaError_t launch_probe_collapse(const double* in, double* out, bool mma, cudaStream_t stream);
}  // namespace tcr

namespace {

using tcr::DevWorkspace;
using tcr::LaunchCfg;

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

struct Config {
    // Defaults = the measured best on B200 at n = 2^30 (profiles/r01/retune_final.txt, profiles/r01/sweep_r01a.jsonl).
    // auto by size (r02 §16): tcgen05 with the dynamic tail for binary16 /
    // fp8 from 512 MiB, mma.sync below and for bfloat16 (resolve_default_algo)
    int default_algo = TCR_ALGO_DEFAULT;
    int blocks_per_sm = 8;
    int unroll = 0;       // 0 = auto: 16 below 2^26 elements, 4 above
    int chain = 4;        // carried chain K (tiles per fp32 accumulator before a flush)
    // tcgen05 (r02): 4 x 32 KiB stages, 4 accumulators with chain 2 = one
    // round per stage (the tight issue loop), CTAs per SM by size (0 = auto)
    int tc05_stages = 4;
    int tc05_stage_kb = 32;
    int tc05_slots = 4;
    int tc05_chain = 2;
    int tc05_ctas = 0;
    int tc05_prefetch = 0;
    int tc05_split = 1;
    int tc05_interleave = 0;
    int tc05_dynamic = 8;  // percent of the chunks handed out at run time (r02 §16)
    int tc05_dyn_min_run = 32;  // ... when every CTA streams >= 32 chunks (r02 §16)
    int rows_tc05 = 1;          // batched rows on tcgen05 where applicable (r02 §17)
    int exact_bulk = 1;         // exact: TMA-fed + dynamic tail from 512 MiB (r02 §18)
    int rows_tc05_stages = 4;
    // bulk (TMA -> SMEM -> mma.sync), r02: one CTA per SM with 4 x 32 KiB
    // (8 tiles per consumer warp per stage = the K = 4 chain per accumulator);
    // 2^30: 0.994-0.995 x mma.sync's time vs 1.07-1.09 x for r01's 6 x 16 KiB,
    // 2 CTAs (profiles/r02/big_n_ab*.txt, bulk_sweep.txt)
    int bulk_stages = 4;
    int bulk_stage_kb = 32;
    int bulk_ctas = 1;
    int exact_unroll = 8;
    int exact_bps = 3;
    int peer_timeout_ms = 10000;
    int pdl = 1;
};
Config g_cfg;
std::mutex g_cfg_mu;

struct DeviceInfo {
    int sms = 0;
    int major = 0;
    int minor = 0;
};

struct Workspace {
    DevWorkspace dev{};
    void* block = nullptr;           // one cudaMalloc for partials + counters
    double* chunk_partials = nullptr;  // host-entry per-chunk fp64 partials
    size_t chunk_cap = 0;
    void* staging[2] = {nullptr, nullptr};
    size_t staging_bytes = 0;
    cudaStream_t copy_stream = nullptr;  // host entry: H2D copies, overlapping the kernels
    cudaEvent_t copied[2] = {nullptr, nullptr};  // staging[b] filled (copy stream)
    cudaEvent_t consumed[2] = {nullptr, nullptr};  // staging[b] read by its kernel (stream)
    cudaEvent_t entry = nullptr;  // the caller's stream position at entry
    float* dev_out = nullptr;
    void* paper_scratch = nullptr;  // study mode: binary16 partials of every level
    size_t paper_scratch_bytes = 0;
};

std::mutex g_mu;
std::map<int, DeviceInfo> g_devices;
std::map<std::pair<int, cudaStream_t>, Workspace*> g_ws;

tcr_status fail(tcr_status s, const char* what) {
    g_last_error = what;
    return s;
}

tcr_status cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? TCR_ERR_OUT_OF_MEMORY : TCR_ERR_CUDA;
}

LaunchCfg make_cfg(const DeviceInfo& di) {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    LaunchCfg c;
    c.sms = di.sms;
    c.blocks_per_sm = g_cfg.blocks_per_sm;
    c.unroll = g_cfg.unroll;
    c.chain = g_cfg.chain;
    c.tc05_stages = g_cfg.tc05_stages;
    c.tc05_stage_kb = g_cfg.tc05_stage_kb;
    c.tc05_slots = g_cfg.tc05_slots;
    c.tc05_chain = g_cfg.tc05_chain;
    c.tc05_ctas = g_cfg.tc05_ctas;
    c.tc05_prefetch = g_cfg.tc05_prefetch;
    c.tc05_split = g_cfg.tc05_split;
    c.tc05_interleave = g_cfg.tc05_interleave;
    c.tc05_dynamic = g_cfg.tc05_dynamic;
    c.tc05_dyn_min_run = g_cfg.tc05_dyn_min_run;
    c.rows_tc05 = g_cfg.rows_tc05;
    c.exact_bulk = g_cfg.exact_bulk;
    c.rows_tc05_stages = g_cfg.rows_tc05_stages;
    c.bulk_stages = g_cfg.bulk_stages;
    c.bulk_stage_kb = g_cfg.bulk_stage_kb;
    c.bulk_ctas = g_cfg.bulk_ctas;
    c.exact_unroll = g_cfg.exact_unroll;
    c.exact_bps = g_cfg.exact_bps;
    c.pdl = g_cfg.pdl;
    return c;
}

// Current device, checked to be compute capability 10.x (B200 = sm_100).
tcr_status current_device(int* dev, DeviceInfo* info) {
    cudaError_t e = cudaGetDevice(dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_devices.find(*dev);
    if (it == g_devices.end()) {
        DeviceInfo di;
        if ((e = cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, *dev)) ||
            (e = cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, *dev)) ||
            (e = cudaDeviceGetAttribute(&di.minor, cudaDevAttrComputeCapabilityMinor, *dev)))
            return cuda_fail(e, "cudaDeviceGetAttribute");
        it = g_devices.emplace(*dev, di).first;
    }
    *info = it->second;
    if (info->major != 10) {
        char buf[128];
        snprintf(buf, sizeof buf, "device %d is sm_%d%d; libtcr is built for sm_100a only",
                 *dev, info->major, info->minor);
        return fail(TCR_ERR_UNSUPPORTED_DEVICE, buf);
    }
    return TCR_OK;
}

// Workspace for (device, stream); partials sized for the largest grid any
// kernel can use on this device (SMs x max CTAs/SM).
tcr_status get_workspace(int dev, const DeviceInfo& di, cudaStream_t stream, Workspace** out) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, stream);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) {
        *out = it->second;
        return TCR_OK;
    }
    auto* ws = new Workspace();
    // 64 doubles per SM: one fp64 partial per CTA for up to 32 CTAs/SM, or
    // the 19-word partials of the exact bfloat16 kernel at 3 CTAs/SM
    const int capacity = di.sms * 64;
    constexpr size_t kCounterBytes = 128;
    const size_t bytes = sizeof(double) * (size_t)capacity + kCounterBytes;
    cudaError_t e = cudaMalloc(&ws->block, bytes);
    if (e != cudaSuccess) {
        delete ws;
        return cuda_fail(e, "cudaMalloc(workspace)");
    }
    char* p = static_cast<char*>(ws->block);
    ws->dev.partials = reinterpret_cast<double*>(p);
    char* ctr = p + sizeof(double) * (size_t)capacity;
    ws->dev.seg_next = reinterpret_cast<unsigned long long*>(ctr);
    ws->dev.seg_exit = reinterpret_cast<unsigned*>(ctr + 8);
    ws->dev.ticket = reinterpret_cast<unsigned*>(ctr + 16);  // kMaxPeers tickets
    ws->dev.chunk_next = reinterpret_cast<unsigned*>(ctr + 64);  // kMaxPeers counters
    ws->dev.capacity = capacity;
    e = cudaMemsetAsync(ctr, 0, kCounterBytes, stream);
    if (e != cudaSuccess) {
        cudaFree(ws->block);
        delete ws;
        return cuda_fail(e, "cudaMemsetAsync(workspace)");
    }
    g_ws.emplace(key, ws);
    *out = ws;
    return TCR_OK;
}

tcr_status prologue(cudaStream_t stream, DeviceInfo* di, Workspace** ws) {
    int dev = 0;
    tcr_status s = current_device(&dev, di);
    if (s != TCR_OK) return s;
    return get_workspace(dev, *di, stream, ws);
}

tcr_status after_launch(cudaError_t e, const char* where, int launches = 1) {
    if (e != cudaSuccess) return cuda_fail(e, where);
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    return TCR_OK;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// TCR_ALGO_DEFAULT resolved for an input of `nbytes` in format `fmt`:
// TCR_CFG_DEFAULT_ALGO unless it is 0 (auto, the default since r02 §16),
// which picks by size -- tcgen05 (TMA ring, one MMA issuer per SM, tight
// issue loop, dynamic tail) for binary16 / fp8 from 512 MiB, where it beats
// mma.sync by 1.5-2.8 % (2^29..2^33, back to back and isolated,
// profiles/r02/tc05_dyn_ab2.txt), mma.sync below (2^24 warm 4.9 vs 6.4 us)
// and for bfloat16 (no dynamic tail: its sums are not multiples of 2^-24).
constexpr size_t kTc05AutoBytes = (size_t)512 << 20;
int resolve_default_algo(size_t nbytes, int fmt) {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    if (g_cfg.default_algo != TCR_ALGO_DEFAULT) return g_cfg.default_algo;
    return (fmt != TCR_DTYPE_BF16 && nbytes >= kTc05AutoBytes) ? TCR_ALGO_TCGEN05 : TCR_ALGO_MMA_SYNC;
}

tcr_status reduce_impl(const tcr_half* x, size_t n, float* out_f32, double* out_f64, int algo,
                       cudaStream_t stream, int fmt = 0) {
    if ((!x && n) || (!out_f32 && !out_f64)) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, fmt >= 2 ? 1 : 2) || (out_f32 && !aligned(out_f32, 4)) ||
        (out_f64 && !aligned(out_f64, 8)))
        return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    if (algo == TCR_ALGO_DEFAULT) algo = resolve_default_algo(n * (fmt >= 2 ? 1u : 2u), fmt);
    if (algo < TCR_ALGO_MMA_SYNC || algo > TCR_ALGO_BULK_MMA)
        return fail(TCR_ERR_INVALID_VALUE, "unknown algo");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue(stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    cudaError_t e;
    if (algo == TCR_ALGO_TCGEN05)
        e = tcr::launch_reduce_tcgen05(fmt, x, n, out_f32, out_f64, ws->dev, cfg, stream);
    else if (algo == TCR_ALGO_BULK_MMA)
        e = tcr::launch_reduce_bulk(fmt, x, n, out_f32, out_f64, ws->dev, cfg, stream);
    else
        e = tcr::launch_reduce_stream(algo == TCR_ALGO_MMA_SYNC, fmt, x, n, out_f32, out_f64, ws->dev,
                                      cfg, stream);
    return after_launch(e, "reduce kernel launch");
}

tcr_status peer_impl(const void* x, size_t n, int dtype, int algo, void* const* mailboxes,
                     int nranks, int rank, float* out_f32, double* out_f64, bool emulate,
                     cudaStream_t stream, bool exact = false, int64_t* out_acc = nullptr) {
    static_assert(tcr::kMailboxBytes == TCR_PEER_MAILBOX_BYTES, "mailbox size");
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    if (algo == TCR_ALGO_DEFAULT) {  // by the per-rank shard size, as reduce_impl
        const size_t es = dtype >= TCR_DTYPE_E4M3 ? 1 : 2;
        algo = resolve_default_algo(n / (size_t)(emulate && nranks > 0 ? nranks : 1) * es, dtype);
        if (algo == TCR_ALGO_BULK_MMA) algo = TCR_ALGO_MMA_SYNC;  // no fused bulk variant
    }
    if (algo != TCR_ALGO_MMA_SYNC && algo != TCR_ALGO_SHUFFLE && algo != TCR_ALGO_TCGEN05)
        return fail(TCR_ERR_INVALID_VALUE,
                    "peer combine algo must be DEFAULT, MMA_SYNC, TCGEN05 or SHUFFLE");
    if (nranks < 1 || nranks > tcr::kMaxPeers || rank < 0 || rank >= nranks)
        return fail(TCR_ERR_INVALID_VALUE, "nranks must be 1..TCR_MAX_PEERS and 0 <= rank < nranks");
    if (!mailboxes || (!x && n) || (!out_f32 && !out_f64 && !out_acc))
        return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (out_acc && !aligned(out_acc, 8)) return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    if (!aligned(x, dtype >= TCR_DTYPE_E4M3 ? 1 : 2) || (out_f32 && !aligned(out_f32, 4)) ||
        (out_f64 && !aligned(out_f64, 8)))
        return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    tcr::PeerCombine pc{};
    for (int r = 0; r < nranks; ++r) {
        if (!mailboxes[r] || !aligned(mailboxes[r], 16))
            return fail(TCR_ERR_INVALID_VALUE, "null or misaligned mailbox");
        pc.mbox[r] = mailboxes[r];
    }
    pc.nranks = nranks;
    pc.rank = rank;
    {
        std::lock_guard<std::mutex> lk(g_cfg_mu);
        pc.timeout_ns = (unsigned long long)g_cfg.peer_timeout_ms * 1000000ull;
    }
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue(stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    if (exact)
        return after_launch(
            tcr::launch_reduce_exact_peer(static_cast<const uint16_t*>(x), n,
                                          reinterpret_cast<long long*>(out_acc), out_f32, out_f64,
                                          ws->dev, cfg, pc, emulate, stream),
            emulate ? "exact peer-emulated launch" : "exact peer launch");
    if (algo == TCR_ALGO_TCGEN05)
        return after_launch(tcr::launch_reduce_tcgen05_peer(dtype, static_cast<const uint16_t*>(x), n,
                                                            out_f32, out_f64, ws->dev, cfg, pc, emulate,
                                                            stream),
                            emulate ? "tcgen05 peer-emulated launch" : "tcgen05 peer launch");
    return after_launch(tcr::launch_reduce_stream_peer(algo == TCR_ALGO_MMA_SYNC, dtype,
                                                       static_cast<const uint16_t*>(x), n, out_f32,
                                                       out_f64, ws->dev, cfg, pc, emulate, stream),
                        emulate ? "peer-emulated reduce launch" : "peer reduce launch");
}

tcr_status segmented_impl(bool mma, bool batched, const void* x, const int64_t* offsets,
                          size_t S, size_t L, float* out, cudaStream_t stream, int fmt = 0) {
    if (!out && S) return fail(TCR_ERR_INVALID_VALUE, "null out");
    if (!batched && !offsets && S) return fail(TCR_ERR_INVALID_VALUE, "null offsets");
    if (!x && S && (batched ? L != 0 : true)) return fail(TCR_ERR_INVALID_VALUE, "null x");
    if (!aligned(x, fmt >= TCR_DTYPE_E4M3 ? 1 : 2) || !aligned(out, 4) || !aligned(offsets, 8))
        return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    if (S == 0) return TCR_OK;
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue(stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    return after_launch(
        tcr::launch_reduce_segmented(mma, fmt, batched, x, offsets, S, L, out, ws->dev, cfg, stream),
        "segmented kernel launch");
}

}  // namespace

extern "C" {

tcr_status tcr_reduce_sum(const tcr_half* x, size_t n, float* out, tcr_stream stream) {
    return reduce_impl(x, n, out, nullptr, TCR_ALGO_DEFAULT, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_shuffle(const tcr_half* x, size_t n, float* out, tcr_stream stream) {
    return reduce_impl(x, n, out, nullptr, TCR_ALGO_SHUFFLE, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_f64(const tcr_half* x, size_t n, double* out, tcr_stream stream) {
    return reduce_impl(x, n, nullptr, out, TCR_ALGO_DEFAULT, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_algo(const tcr_half* x, size_t n, float* out_f32, double* out_f64,
                               tcr_algo algo, tcr_stream stream) {
    return reduce_impl(x, n, out_f32, out_f64, (int)algo, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_ex(const void* x, size_t n, tcr_dtype dtype, float* out_f32,
                             double* out_f64, tcr_algo algo, tcr_stream stream) {
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    return reduce_impl(static_cast<const tcr_half*>(x), n, out_f32, out_f64, (int)algo,
                       (cudaStream_t)stream, (int)dtype);
}

tcr_status tcr_reduce_sum_segmented_ex(const void* x, tcr_dtype dtype, const int64_t* offsets,
                                       size_t num_segments, float* out, tcr_algo algo,
                                       tcr_stream stream) {
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    if (algo != TCR_ALGO_DEFAULT && algo != TCR_ALGO_MMA_SYNC && algo != TCR_ALGO_SHUFFLE)
        return fail(TCR_ERR_INVALID_VALUE, "segmented algo must be DEFAULT, MMA_SYNC or SHUFFLE");
    return segmented_impl(algo != TCR_ALGO_SHUFFLE, false, x, offsets, num_segments, 0, out,
                          (cudaStream_t)stream, (int)dtype);
}

tcr_status tcr_reduce_sum_batched_ex(const void* x, tcr_dtype dtype, size_t num_segments,
                                     size_t segment_len, float* out, tcr_algo algo,
                                     tcr_stream stream) {
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    if (algo != TCR_ALGO_DEFAULT && algo != TCR_ALGO_MMA_SYNC && algo != TCR_ALGO_SHUFFLE)
        return fail(TCR_ERR_INVALID_VALUE, "batched algo must be DEFAULT, MMA_SYNC or SHUFFLE");
    return segmented_impl(algo != TCR_ALGO_SHUFFLE, true, x, nullptr, num_segments, segment_len, out,
                          (cudaStream_t)stream, (int)dtype);
}

tcr_status tcr_reduce_sum_segmented(const tcr_half* x, const int64_t* offsets,
                                    size_t num_segments, float* out, tcr_stream stream) {
    return segmented_impl(true, false, x, offsets, num_segments, 0, out, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_segmented_shuffle(const tcr_half* x, const int64_t* offsets,
                                            size_t num_segments, float* out, tcr_stream stream) {
    return segmented_impl(false, false, x, offsets, num_segments, 0, out, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_batched(const tcr_half* x, size_t num_segments, size_t segment_len,
                                  float* out, tcr_stream stream) {
    return segmented_impl(true, true, x, nullptr, num_segments, segment_len, out,
                          (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_batched_shuffle(const tcr_half* x, size_t num_segments,
                                          size_t segment_len, float* out, tcr_stream stream) {
    return segmented_impl(false, true, x, nullptr, num_segments, segment_len, out,
                          (cudaStream_t)stream);
}

// End-to-end host entry for any input type: chunks of 128 MiB of input bytes
// through two staging buffers.  The H2D copies run on the workspace's copy
// stream and the kernels on the caller's stream; events order each buffer's
// reuse (copy c+2 waits for kernel c), so the H2D of chunk c+1 overlaps the
// kernel of chunk c (with pinned host memory; pageable memory serialises in
// the driver).  Kernels use the library's default algorithm for the type.
static tcr_status reduce_host_impl(const void* x, size_t n, int fmt, float* out,
                                   cudaStream_t stream) {
    const size_t es = fmt >= TCR_DTYPE_E4M3 ? 1 : 2;
    if ((!x && n) || !out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, es)) return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue(stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    const size_t kChunk = ((size_t)1 << 27) / es;  // elements per staged chunk (128 MiB)
    const size_t chunks = n ? (n + kChunk - 1) / kChunk : 0;
    cudaError_t e;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!ws->dev_out && (e = cudaMalloc(&ws->dev_out, sizeof(float))))
            return cuda_fail(e, "cudaMalloc(out)");
        if (ws->chunk_cap < chunks || !ws->chunk_partials) {
            if (ws->chunk_partials) cudaFree(ws->chunk_partials);
            ws->chunk_partials = nullptr;
            const size_t cap = chunks < 64 ? 64 : chunks;
            if ((e = cudaMalloc(&ws->chunk_partials, cap * sizeof(double))))
                return cuda_fail(e, "cudaMalloc(chunk partials)");
            ws->chunk_cap = cap;
        }
        const size_t need = (n < kChunk ? (n ? n : 1) : kChunk) * es;
        if (ws->staging_bytes < need) {
            for (void*& b : ws->staging) {
                if (b) cudaFree(b);
                b = nullptr;
            }
            for (void*& b : ws->staging)
                if ((e = cudaMalloc(&b, need))) return cuda_fail(e, "cudaMalloc(staging)");
            ws->staging_bytes = need;
        }
        if (!ws->copy_stream) {
            if ((e = cudaStreamCreateWithFlags(&ws->copy_stream, cudaStreamNonBlocking)))
                return cuda_fail(e, "cudaStreamCreate(copy)");
            for (int b = 0; b < 2; ++b)
                if ((e = cudaEventCreateWithFlags(&ws->copied[b], cudaEventDisableTiming)) ||
                    (e = cudaEventCreateWithFlags(&ws->consumed[b], cudaEventDisableTiming)))
                    return cuda_fail(e, "cudaEventCreate");
            if ((e = cudaEventCreateWithFlags(&ws->entry, cudaEventDisableTiming)))
                return cuda_fail(e, "cudaEventCreate");
        }
    }
    int launches = 0;
    const char* xb = static_cast<const char*>(x);
    // the copy stream starts after the caller's earlier work (staging reuse
    // across calls, and the caller's ordering of x)
    if ((e = cudaEventRecord(ws->entry, stream)) ||
        (e = cudaStreamWaitEvent(ws->copy_stream, ws->entry, 0)))
        return cuda_fail(e, "event ordering");
    for (size_t c = 0; c < chunks; ++c) {
        const size_t lo = c * kChunk, cnt = (n - lo < kChunk) ? n - lo : kChunk;
        const int b = (int)(c & 1);
        void* buf = ws->staging[b];
        if (c >= 2 && (e = cudaStreamWaitEvent(ws->copy_stream, ws->consumed[b], 0)))
            return cuda_fail(e, "cudaStreamWaitEvent(consumed)");
        if ((e = cudaMemcpyAsync(buf, xb + lo * es, cnt * es, cudaMemcpyHostToDevice,
                                 ws->copy_stream)))
            return cuda_fail(e, "cudaMemcpyAsync(H2D)");
        if ((e = cudaEventRecord(ws->copied[b], ws->copy_stream)) ||
            (e = cudaStreamWaitEvent(stream, ws->copied[b], 0)))
            return cuda_fail(e, "event ordering (copied)");
        const uint16_t* db = static_cast<const uint16_t*>(buf);
        // the default algorithm for this chunk's size (reduce_impl's rule)
        const int a = resolve_default_algo(cnt * es, fmt);
        if (a == TCR_ALGO_TCGEN05)
            e = tcr::launch_reduce_tcgen05(fmt, db, cnt, nullptr, ws->chunk_partials + c, ws->dev,
                                           cfg, stream);
        else if (a == TCR_ALGO_BULK_MMA)
            e = tcr::launch_reduce_bulk(fmt, db, cnt, nullptr, ws->chunk_partials + c, ws->dev, cfg,
                                        stream);
        else
            e = tcr::launch_reduce_stream(a == TCR_ALGO_MMA_SYNC, fmt, db, cnt, nullptr,
                                          ws->chunk_partials + c, ws->dev, cfg, stream);
        if (e) return cuda_fail(e, "reduce kernel launch");
        if ((e = cudaEventRecord(ws->consumed[b], stream)))
            return cuda_fail(e, "cudaEventRecord(consumed)");
        ++launches;
    }
    if ((e = tcr::launch_sum_partials(ws->chunk_partials, chunks, ws->dev_out, nullptr, stream)))
        return cuda_fail(e, "sum_partials launch");
    ++launches;
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    if ((e = cudaMemcpyAsync(out, ws->dev_out, sizeof(float), cudaMemcpyDeviceToHost, stream)))
        return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    if ((e = cudaStreamSynchronize(stream))) return cuda_fail(e, "cudaStreamSynchronize");
    return TCR_OK;
}

tcr_status tcr_reduce_sum_host(const tcr_half* x, size_t n, float* out, tcr_stream stream) {
    return reduce_host_impl(x, n, TCR_DTYPE_F16, out, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_host_ex(const void* x, size_t n, tcr_dtype dtype, float* out,
                                  tcr_stream stream) {
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    return reduce_host_impl(x, n, (int)dtype, out, (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_exact(const tcr_half* x, size_t n, int64_t* acc, float* out_f32,
                                double* out_f64, tcr_stream stream) {
    if ((!x && n) || (!acc && !out_f32 && !out_f64))
        return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, 2) || !aligned(acc, 8) || !aligned(out_f32, 4) || !aligned(out_f64, 8))
        return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue((cudaStream_t)stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    return after_launch(tcr::launch_reduce_exact(0, x, n, reinterpret_cast<long long*>(acc), out_f32,
                                                 out_f64, ws->dev, cfg, (cudaStream_t)stream),
                        "exact kernel launch");
}

tcr_status tcr_reduce_sum_exact_ex(const void* x, size_t n, tcr_dtype dtype, int64_t* acc,
                                   float* out_f32, double* out_f64, tcr_stream stream) {
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    if ((!x && n) || (!acc && !out_f32 && !out_f64))
        return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, dtype <= TCR_DTYPE_BF16 ? 2 : 1) || !aligned(acc, 8) || !aligned(out_f32, 4) ||
        !aligned(out_f64, 8))
        return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue((cudaStream_t)stream, &di, &ws);
    if (s != TCR_OK) return s;
    const LaunchCfg cfg = make_cfg(di);
    if (dtype == TCR_DTYPE_BF16)
        return after_launch(tcr::launch_reduce_exact_bf16(static_cast<const uint16_t*>(x), n,
                                                          reinterpret_cast<long long*>(acc), out_f32,
                                                          out_f64, ws->dev, cfg, (cudaStream_t)stream),
                            "exact bf16 kernel launch");
    if (dtype == TCR_DTYPE_E4M3 && tcr::exact_e4m3_tc05_applies(n, cfg)) {
        int launches = 1;
        const cudaError_t e = tcr::launch_exact_e4m3_tc05(static_cast<const uint8_t*>(x), n,
                                                          reinterpret_cast<long long*>(acc), out_f32,
                                                          out_f64, ws->dev, cfg, (cudaStream_t)stream,
                                                          &launches);
        return after_launch(e, "exact E4M3 (tcgen05) launch", launches);
    }
    return after_launch(tcr::launch_reduce_exact((int)dtype, x, n, reinterpret_cast<long long*>(acc),
                                                 out_f32, out_f64, ws->dev, cfg, (cudaStream_t)stream),
                        "exact kernel launch");
}

tcr_status tcr_exact_finalize(const int64_t* acc, float* out_f32, double* out_f64,
                              tcr_stream stream) {
    if (!acc || (!out_f32 && !out_f64)) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    return after_launch(tcr::launch_exact_finalize(reinterpret_cast<const long long*>(acc),
                                                   out_f32, out_f64, (cudaStream_t)stream),
                        "exact finalize launch");
}

tcr_status tcr_exact_finalize_ex(const int64_t* acc, tcr_dtype dtype, float* out_f32,
                                 double* out_f64, tcr_stream stream) {
    if (!acc || (!out_f32 && !out_f64)) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (dtype < TCR_DTYPE_F16 || dtype > TCR_DTYPE_E5M2)
        return fail(TCR_ERR_INVALID_VALUE, "unknown dtype");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    const long long* a = reinterpret_cast<const long long*>(acc);
    return after_launch(dtype == TCR_DTYPE_BF16
                            ? tcr::launch_exact_bf16_finalize(a, out_f32, out_f64, (cudaStream_t)stream)
                            : tcr::launch_exact_finalize(a, out_f32, out_f64, (cudaStream_t)stream),
                        "exact finalize launch");
}

tcr_status tcr_round_f64_to_f32(const double* in, float* out, tcr_stream stream) {
    if (!in || !out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    return after_launch(tcr::launch_round_f64(in, out, (cudaStream_t)stream), "round launch");
}

tcr_status tcr_probe_mma(const tcr_half* a, const float* c, float* d, tcr_algo algo,
                         tcr_stream stream) {
    if (!a || !c || !d) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    if (algo == TCR_ALGO_MMA_SYNC)
        return after_launch(tcr::launch_probe_mma_sync(a, c, d, (cudaStream_t)stream), "probe");
    if (algo == TCR_ALGO_TCGEN05)
        return after_launch(tcr::launch_probe_mma_tcgen05(a, c, d, (cudaStream_t)stream),
                            "probe");
    return fail(TCR_ERR_INVALID_VALUE, "probe algo must be MMA_SYNC or TCGEN05");
}

tcr_status tcr_reduce_sum_peer(const void* x, size_t n, tcr_dtype dtype, tcr_algo algo,
                               void* const* mailboxes, int nranks, int rank, float* out_f32,
                               double* out_f64, tcr_stream stream) {
    return peer_impl(x, n, (int)dtype, (int)algo, mailboxes, nranks, rank, out_f32, out_f64, false,
                     (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_peer_emulated(const void* x, size_t n, tcr_dtype dtype, tcr_algo algo,
                                        void* const* mailboxes, int nranks, float* out_f32,
                                        double* out_f64, tcr_stream stream) {
    return peer_impl(x, n, (int)dtype, (int)algo, mailboxes, nranks, 0, out_f32, out_f64, true,
                     (cudaStream_t)stream);
}

tcr_status tcr_reduce_sum_exact_peer(const tcr_half* x, size_t n, void* const* mailboxes,
                                     int nranks, int rank, int64_t* acc, float* out_f32,
                                     double* out_f64, tcr_stream stream) {
    return peer_impl(x, n, TCR_DTYPE_F16, TCR_ALGO_DEFAULT, mailboxes, nranks, rank, out_f32,
                     out_f64, false, (cudaStream_t)stream, true, acc);
}

tcr_status tcr_reduce_sum_exact_peer_emulated(const tcr_half* x, size_t n,
                                              void* const* mailboxes, int nranks, int64_t* acc,
                                              float* out_f32, double* out_f64, tcr_stream stream) {
    return peer_impl(x, n, TCR_DTYPE_F16, TCR_ALGO_DEFAULT, mailboxes, nranks, 0, out_f32, out_f64,
                     true, (cudaStream_t)stream, true, acc);
}

tcr_status tcr_peer_mailbox_alloc(void** mailbox) {
    if (!mailbox) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, tcr::kMailboxBytes);  // plain cudaMalloc: IPC-exportable
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(mailbox)");
    if ((e = cudaMemset(p, 0, tcr::kMailboxBytes))) {
        cudaFree(p);
        return cuda_fail(e, "cudaMemset(mailbox)");
    }
    *mailbox = p;
    return TCR_OK;
}

tcr_status tcr_peer_mailbox_free(void* mailbox) {
    if (!mailbox) return TCR_OK;
    cudaError_t e = cudaFree(mailbox);
    return e == cudaSuccess ? TCR_OK : cuda_fail(e, "cudaFree(mailbox)");
}

tcr_status tcr_peer_mailbox_reset(void* mailbox, tcr_stream stream) {
    if (!mailbox) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    cudaError_t e = cudaMemsetAsync(mailbox, 0, tcr::kMailboxBytes, (cudaStream_t)stream);
    return e == cudaSuccess ? TCR_OK : cuda_fail(e, "cudaMemsetAsync(mailbox)");
}

tcr_status tcr_peer_mailbox_error(const void* mailbox, int* timed_out) {
    if (!mailbox || !timed_out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    unsigned w = 0;
    cudaError_t e = cudaMemcpy(&w, static_cast<const char*>(mailbox) + tcr::kMailboxErrOffset,
                               sizeof w, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(mailbox error)");
    *timed_out = w ? 1 : 0;
    return TCR_OK;
}

tcr_status tcr_peer_ipc_handle(const void* mailbox, void* handle) {
    if (!mailbox || !handle) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == TCR_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(mailbox));
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    memcpy(handle, &h, sizeof h);
    return TCR_OK;
}

tcr_status tcr_peer_ipc_open(const void* handle, void** peer_mailbox) {
    if (!handle || !peer_mailbox) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *peer_mailbox = p;
    return TCR_OK;
}

tcr_status tcr_peer_ipc_close(void* peer_mailbox) {
    if (!peer_mailbox) return TCR_OK;
    cudaError_t e = cudaIpcCloseMemHandle(peer_mailbox);
    return e == cudaSuccess ? TCR_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

tcr_status tcr_reduce_sum_paper_f16(const tcr_half* x, size_t n, float* out, tcr_stream stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if ((!x && n) || !out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, 2) || !aligned(out, 4)) return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue(stream, &di, &ws);
    if (s != TCR_OK) return s;
    const size_t need = tcr::paper_scratch_elems(n) * sizeof(uint16_t) + 16;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (ws->paper_scratch_bytes < need) {  // grows once per stream, never shrinks
            if (ws->paper_scratch) cudaFree(ws->paper_scratch);
            ws->paper_scratch = nullptr;
            ws->paper_scratch_bytes = 0;
            cudaError_t e = cudaMalloc(&ws->paper_scratch, need);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(paper scratch)");
            ws->paper_scratch_bytes = need;
        }
    }
    int launches = 0;
    cudaError_t e = tcr::launch_reduce_paper_f16(x, n, static_cast<uint16_t*>(ws->paper_scratch), out,
                                                 di.sms, stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "paper-mode launch");
    g_launches.fetch_add(launches, std::memory_order_relaxed);
    return TCR_OK;
}

tcr_status tcr_reduce_sum_study_fp32(const tcr_half* x, size_t n, int kahan, float* out,
                                     tcr_stream stream) {
    if ((!x && n) || !out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (!aligned(x, 2) || !aligned(out, 4)) return fail(TCR_ERR_INVALID_VALUE, "misaligned pointer");
    DeviceInfo di;
    Workspace* ws = nullptr;
    tcr_status s = prologue((cudaStream_t)stream, &di, &ws);
    if (s != TCR_OK) return s;
    return after_launch(tcr::launch_study_fp32(x, n, kahan != 0, out, ws->dev, di.sms,
                                               (cudaStream_t)stream),
                        "study fp32 launch");
}

tcr_status tcr_probe_collapse(const double* in, double* out, tcr_algo algo, tcr_stream stream) {
    if (!in || !out) return fail(TCR_ERR_INVALID_VALUE, "null pointer");
    if (algo != TCR_ALGO_MMA_SYNC && algo != TCR_ALGO_SHUFFLE)
        return fail(TCR_ERR_INVALID_VALUE, "collapse probe algo must be MMA_SYNC or SHUFFLE");
    DeviceInfo di;
    int dev;
    tcr_status s = current_device(&dev, &di);
    if (s != TCR_OK) return s;
    return after_launch(tcr::launch_probe_collapse(in, out, algo == TCR_ALGO_MMA_SYNC,
                                                   (cudaStream_t)stream),
                        "collapse probe");
}

tcr_status tcr_set_config(tcr_config_key key, int value) {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    switch (key) {
        case TCR_CFG_DEFAULT_ALGO:  // 0 = auto by input size
            if (value < TCR_ALGO_DEFAULT || value > TCR_ALGO_BULK_MMA) break;
            g_cfg.default_algo = value;
            return TCR_OK;
        case TCR_CFG_BLOCKS_PER_SM:
            if (value < 1 || value > 32) break;
            g_cfg.blocks_per_sm = value;
            return TCR_OK;
        case TCR_CFG_UNROLL:
            if (value != 0 && value != 4 && value != 8 && value != 16) break;
            g_cfg.unroll = value;
            return TCR_OK;
        case TCR_CFG_TC05_STAGES:
            if (value < 2 || value > 16) break;
            g_cfg.tc05_stages = value;
            return TCR_OK;
        case TCR_CFG_TC05_STAGE_KB:
            if (value < 4 || value > 64 || value % 4) break;
            g_cfg.tc05_stage_kb = value;
            return TCR_OK;
        case TCR_CFG_CHAIN:
            if (value < 1 || value > 1024) break;
            g_cfg.chain = value;
            return TCR_OK;
        case TCR_CFG_TC05_SLOTS:
            if (value < 1 || value > 16 || (value & (value - 1))) break;
            g_cfg.tc05_slots = value;
            return TCR_OK;
        case TCR_CFG_TC05_CHAIN:
            if (value < 1 || value > 256) break;
            g_cfg.tc05_chain = value;
            return TCR_OK;
        case TCR_CFG_TC05_CTAS_PER_SM:
            if (value < 0 || value > 4) break;  // 0 = auto by input size
            g_cfg.tc05_ctas = value;
            return TCR_OK;
        case TCR_CFG_TC05_PREFETCH:
            if (value < 0 || value > 64) break;
            g_cfg.tc05_prefetch = value;
            return TCR_OK;
        case TCR_CFG_TC05_SPLIT:
            if (value != 1 && value != 2 && value != 4 && value != 8) break;
            g_cfg.tc05_split = value;
            return TCR_OK;
        case TCR_CFG_TC05_INTERLEAVE:
            if (value != 0 && value != 1) break;
            g_cfg.tc05_interleave = value;
            return TCR_OK;
        case TCR_CFG_TC05_DYNAMIC:
            if (value < 0 || value > 100) break;
            g_cfg.tc05_dynamic = value;
            return TCR_OK;
        case TCR_CFG_TC05_DYN_MIN_RUN:
            if (value < 0 || value > 1 << 20) break;
            g_cfg.tc05_dyn_min_run = value;
            return TCR_OK;
        case TCR_CFG_EXACT_BULK:
            if (value < 0 || value > 2) break;
            g_cfg.exact_bulk = value;
            return TCR_OK;
        case TCR_CFG_ROWS_TC05:
            if (value != 0 && value != 1) break;
            g_cfg.rows_tc05 = value;
            return TCR_OK;
        case TCR_CFG_ROWS_TC05_STAGES:
            if (value < 2 || value > 6) break;
            g_cfg.rows_tc05_stages = value;
            return TCR_OK;
        case TCR_CFG_BULK_STAGES:
            if (value < 2 || value > 32) break;
            g_cfg.bulk_stages = value;
            return TCR_OK;
        case TCR_CFG_BULK_STAGE_KB:
            if (value < 4 || value > 64 || value % 4) break;
            g_cfg.bulk_stage_kb = value;
            return TCR_OK;
        case TCR_CFG_BULK_CTAS_PER_SM:
            if (value < 1 || value > 8) break;
            g_cfg.bulk_ctas = value;
            return TCR_OK;
        case TCR_CFG_EXACT_UNROLL:
            if (value != 4 && value != 8) break;
            g_cfg.exact_unroll = value;
            return TCR_OK;
        case TCR_CFG_EXACT_BLOCKS_PER_SM:
            if (value < 1 || value > 8) break;
            g_cfg.exact_bps = value;
            return TCR_OK;
        case TCR_CFG_PDL:
            if (value < 0 || value > 1) break;
            g_cfg.pdl = value;
            return TCR_OK;
        case TCR_CFG_PEER_TIMEOUT_MS:
            if (value < 1 || value > 600000) break;
            g_cfg.peer_timeout_ms = value;
            return TCR_OK;
    }
    g_last_error = "invalid config key or value";
    return TCR_ERR_INVALID_VALUE;
}

int tcr_get_config(tcr_config_key key) {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    switch (key) {
        case TCR_CFG_DEFAULT_ALGO: return g_cfg.default_algo;
        case TCR_CFG_BLOCKS_PER_SM: return g_cfg.blocks_per_sm;
        case TCR_CFG_UNROLL: return g_cfg.unroll;
        case TCR_CFG_TC05_STAGES: return g_cfg.tc05_stages;
        case TCR_CFG_TC05_STAGE_KB: return g_cfg.tc05_stage_kb;
        case TCR_CFG_CHAIN: return g_cfg.chain;
        case TCR_CFG_TC05_SLOTS: return g_cfg.tc05_slots;
        case TCR_CFG_TC05_CHAIN: return g_cfg.tc05_chain;
        case TCR_CFG_TC05_CTAS_PER_SM: return g_cfg.tc05_ctas;
        case TCR_CFG_TC05_PREFETCH: return g_cfg.tc05_prefetch;
        case TCR_CFG_TC05_SPLIT: return g_cfg.tc05_split;
        case TCR_CFG_TC05_INTERLEAVE: return g_cfg.tc05_interleave;
        case TCR_CFG_TC05_DYNAMIC: return g_cfg.tc05_dynamic;
        case TCR_CFG_TC05_DYN_MIN_RUN: return g_cfg.tc05_dyn_min_run;
        case TCR_CFG_ROWS_TC05: return g_cfg.rows_tc05;
        case TCR_CFG_EXACT_BULK: return g_cfg.exact_bulk;
        case TCR_CFG_ROWS_TC05_STAGES: return g_cfg.rows_tc05_stages;
        case TCR_CFG_BULK_STAGES: return g_cfg.bulk_stages;
        case TCR_CFG_BULK_STAGE_KB: return g_cfg.bulk_stage_kb;
        case TCR_CFG_BULK_CTAS_PER_SM: return g_cfg.bulk_ctas;
        case TCR_CFG_EXACT_UNROLL: return g_cfg.exact_unroll;
        case TCR_CFG_EXACT_BLOCKS_PER_SM: return g_cfg.exact_bps;
        case TCR_CFG_PEER_TIMEOUT_MS: return g_cfg.peer_timeout_ms;
        case TCR_CFG_PDL: return g_cfg.pdl;
    }
    return -1;
}

const char* tcr_status_string(tcr_status s) {
    switch (s) {
        case TCR_OK: return "TCR_OK";
        case TCR_ERR_INVALID_VALUE: return "TCR_ERR_INVALID_VALUE";
        case TCR_ERR_UNSUPPORTED_DEVICE: return "TCR_ERR_UNSUPPORTED_DEVICE";
        case TCR_ERR_OUT_OF_MEMORY: return "TCR_ERR_OUT_OF_MEMORY";
        case TCR_ERR_CUDA: return "TCR_ERR_CUDA";
    }
    return "TCR_ERR_UNKNOWN";
}

const char* tcr_last_error(void) { return g_last_error.c_str(); }

tcr_status tcr_release_workspaces(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_ws) {
        Workspace* ws = kv.second;
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(kv.first.first);
        cudaFree(ws->block);
        if (ws->chunk_partials) cudaFree(ws->chunk_partials);
        for (void* b : ws->staging)
            if (b) cudaFree(b);
        if (ws->copy_stream) {
            for (int b = 0; b < 2; ++b) {
                cudaEventDestroy(ws->copied[b]);
                cudaEventDestroy(ws->consumed[b]);
            }
            cudaEventDestroy(ws->entry);
            cudaStreamDestroy(ws->copy_stream);
        }
        if (ws->dev_out) cudaFree(ws->dev_out);
        if (ws->paper_scratch) cudaFree(ws->paper_scratch);
        cudaSetDevice(prev);
        delete ws;
    }
    g_ws.clear();
    return TCR_OK;
}

uint64_t tcr_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

tcr_algo tcr_default_algo(size_t n, tcr_dtype dtype) {
    const size_t es = (dtype == TCR_DTYPE_E4M3 || dtype == TCR_DTYPE_E5M2) ? 1 : 2;
    return (tcr_algo)resolve_default_algo(n * es, (int)dtype);
}

int tcr_version(void) { return TCR_VERSION; }

}  // extern "C"
