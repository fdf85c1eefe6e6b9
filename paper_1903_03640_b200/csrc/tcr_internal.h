// tcr_internal.h -- host-side declarations shared by the API and the kernel
// translation units of libtcr (not part of the public ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tcr {

// Library-owned per-(device, stream) workspace, passed by value to kernels.
struct DevWorkspace {
    double* partials;               // [capacity] fp64 partial of every CTA (level >= 3)
    unsigned* ticket;               // last-CTA completion ticket (self-resetting); kMaxPeers
                                    // consecutive tickets (one per emulated rank)
    unsigned long long* seg_next;   // segmented: next segment index (self-resetting)
    unsigned* seg_exit;             // segmented: warps that finished (self-resetting)
    unsigned* chunk_next;           // tcgen05 dynamic tail: next chunk ticket (self-resetting);
                                    // kMaxPeers consecutive counters (one per emulated rank)
    int capacity;                   // entries in partials
};

// NEXT-2 fused cross-GPU combine (tcr_peer.cuh).  A mailbox is a small
// device allocation on every rank; slot [parity][src] of rank d's mailbox
// receives src's fp64 partial for the epoch of that parity.
constexpr int kMaxPeers = 8;           // ranks per peer group (one NVLink node)
constexpr int kMailboxBytes = 2048;    // fp64 slots, error word, epoch, exact slots
constexpr int kMailboxErrOffset = 256; // uint32: set to 1 when a wait timed out
constexpr int kMailboxEpochOffset = 264;  // uint64: combines completed by the owning rank
constexpr int kMailboxExactOffset = 512;  // 2 x kMaxPeers x 96 B exact-limb slots

struct PeerCombine {
    void* mbox[kMaxPeers];        // mailbox of every rank (own + mapped peers), by rank
    int nranks;                   // 0 = no combine (single-GPU result)
    int rank;                     // this process's rank (emulation: base rank 0)
    unsigned long long timeout_ns;  // bound on the wait for the peers' partials
};

struct LaunchCfg {
    int sms;            // SM count of the device
    int blocks_per_sm;  // CTAs per SM for the streaming kernels
    int unroll;         // 16-byte loads in flight per lane (4, 8 or 16)
    int chain;          // carried chain K in tiles (mma_sync / shuffle); the kernel
                        // flushes every max(1, 2K/unroll) iterations of `unroll` tiles
    int tc05_stages;    // tcgen05 kernel: SMEM ring stages
    int tc05_stage_kb;  // tcgen05 kernel: KiB per stage (multiple of 4)
    int tc05_slots;     // tcgen05 kernel: independent accumulators per TMEM buffer
    int tc05_chain;     // tcgen05 kernel: MMAs carried per accumulator before a flush
    int tc05_ctas;      // tcgen05 kernel: CTAs per SM
    int tc05_prefetch;  // tcgen05 kernel: L2 prefetch distance in chunks
    int tc05_split;     // tcgen05 kernel: bulk copies per stage
    int tc05_interleave;  // tcgen05 kernel: chunk-to-CTA mapping (0 contiguous, 1 interleaved)
    int tc05_dynamic;     // tcgen05 kernel: percent of the chunks handed out at run time
                          // (dynamic tail; 0 = static partition)
    int tc05_dyn_min_run; // tcgen05 kernel: the dynamic tail only when every CTA's
                          // static run would be at least this many chunks
    int exact_bulk;       // exact: 1 = TMA-fed kernel + dynamic tail, binary16 from 128 MiB (2: always)
    int rows_tc05;        // batched: 1 = fixed-length rows on tcgen05 (128 segments per MMA)
    int rows_tc05_stages; // batched tcgen05 kernel: SMEM ring stages of 16 KiB
    int bulk_stages;      // bulk (TMA -> SMEM -> mma.sync) kernel: ring stages
    int bulk_stage_kb;    // bulk kernel: KiB per stage (multiple of 4)
    int bulk_ctas;        // bulk kernel: CTAs per SM
    int exact_unroll;     // exact kernel: 16-byte loads in flight per lane (4 or 8)
    int exact_bps;        // exact kernel: CTAs per SM
    int pdl;              // streaming kernels: programmatic dependent launch (0 / 1)
};

// Each launcher enqueues exactly one kernel on `stream` and returns the
// cudaGetLastError() of the launch.
// fmt: 0 binary16, 1 bfloat16, 2 fp8 E4M3, 3 fp8 E5M2 (n counts elements)
cudaError_t launch_reduce_stream(bool mma, int fmt, const uint16_t* x, size_t n, float* out_f32,
                                 double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                 cudaStream_t stream);
// Flat reduction fused with the cross-GPU combine (NEXT-2).  emulate = false:
// one rank of a real peer group (pc.rank); emulate = true: ONE cooperative
// launch whose grid.y slices are pc.nranks emulated ranks, slice r reducing
// the shard [r n / P, (r+1) n / P) of x and writing out_*[r].
cudaError_t launch_reduce_stream_peer(bool mma, int fmt, const uint16_t* x, size_t n,
                                      float* out_f32, double* out_f64, const DevWorkspace& ws,
                                      const LaunchCfg& cfg, const PeerCombine& pc, bool emulate,
                                      cudaStream_t stream);
cudaError_t launch_reduce_tcgen05(int fmt, const uint16_t* x, size_t n, float* out_f32,
                                  double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                  cudaStream_t stream);
// NEXT-2 on the tcgen05 kernel: the cross-GPU combine fused into its last CTA
// (emulate: nranks grid slices in one cooperative launch)
cudaError_t launch_reduce_tcgen05_peer(int fmt, const uint16_t* x, size_t n, float* out_f32,
                                       double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                       const PeerCombine& pc, bool emulate, cudaStream_t stream);
cudaError_t launch_reduce_segmented(bool mma, int fmt, bool batched, const void* x,
                                    const int64_t* offsets, size_t num_segments,
                                    size_t segment_len, float* out, const DevWorkspace& ws,
                                    const LaunchCfg& cfg, cudaStream_t stream);
cudaError_t launch_reduce_bulk(int fmt, const uint16_t* x, size_t n, float* out_f32,
                               double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                               cudaStream_t stream);
cudaError_t launch_reduce_exact(int fmt, const void* x, size_t n, long long* out_acc,
                                float* out_f32, double* out_f64, const DevWorkspace& ws,
                                const LaunchCfg& cfg, cudaStream_t stream);
// Exact reduction of bfloat16 (tcr_exact_bf16.cu): 8 exponent windows.
// out_acc: 27 int64 (8 windows x 3 limbs, 3 special counts), integer-summable.
cudaError_t launch_reduce_exact_bf16(const uint16_t* x, size_t n, long long* out_acc,
                                     float* out_f32, double* out_f64, const DevWorkspace& ws,
                                     const LaunchCfg& cfg, cudaStream_t stream);
cudaError_t launch_exact_bf16_finalize(const long long* acc, float* out_f32, double* out_f64,
                                       cudaStream_t stream);
// Exact reduction fused with the cross-GPU combine of the int64 limbs
// (NEXT-2 x NEXT-3); emulate as for launch_reduce_stream_peer (out_acc: 6
// words per rank, out_f32 / out_f64: one per rank).
cudaError_t launch_reduce_exact_peer(const uint16_t* x, size_t n, long long* out_acc,
                                     float* out_f32, double* out_f64, const DevWorkspace& ws,
                                     const LaunchCfg& cfg, const PeerCombine& pc, bool emulate,
                                     cudaStream_t stream);
cudaError_t launch_exact_finalize(const long long* acc, float* out_f32, double* out_f64,
                                  cudaStream_t stream);
// Exact fp8 E4M3 on the tcgen05 dynamic-tail kernel (r02 §16: its rows of 64
// E4M3 values are exact in binary32) + a NaN count when needed; *launches =
// the kernels enqueued (1, or 2 with out_acc).
bool exact_e4m3_tc05_applies(size_t n, const LaunchCfg& cfg);
cudaError_t launch_exact_e4m3_tc05(const uint8_t* x, size_t n, long long* out_acc, float* out_f32,
                                   double* out_f64, const DevWorkspace& ws, const LaunchCfg& cfg,
                                   cudaStream_t stream, int* launches);
// The paper's algorithm literally (study mode, tcr_paper.cu): fp16 MMAs, fp16
// partials in `scratch` (paper_scratch_elems(n) binary16), one launch per level.
size_t paper_scratch_elems(size_t n);
cudaError_t launch_reduce_paper_f16(const uint16_t* x, size_t n, uint16_t* scratch, float* out_f32,
                                    int sms, cudaStream_t stream, int* launches);
// Study mode (NEXT-1): the classic reduction entirely in binary32, naive or
// Kahan-compensated (lane and grid levels).
cudaError_t launch_study_fp32(const uint16_t* x, size_t n, bool kahan, float* out,
                              const DevWorkspace& ws, int sms, cudaStream_t stream);
cudaError_t launch_sum_partials(const double* partials, size_t count, float* out_f32,
                                double* out_f64, cudaStream_t stream);
cudaError_t launch_round_f64(const double* in, float* out, cudaStream_t stream);
cudaError_t launch_probe_mma(int algo, const uint16_t* a, const float* c, float* d,
                             cudaStream_t stream);

// Grid size of the streaming kernels for n elements (shared by the API's
// workspace sizing and the launchers).
int stream_grid(size_t n, const LaunchCfg& cfg, int resident = 0);
// Batched fixed-length rows on tcgen05 (tcr_rows_tc05.cu): 128 segments as
// the 128 rows of A, TMA tensor copies with 128-byte swizzle.
bool rows_tc05_supported(int fmt, const void* x, size_t S, size_t L);
cudaError_t launch_reduce_rows_tc05(int fmt, const void* x, size_t S, size_t L, float* out,
                                    const DevWorkspace& ws, const LaunchCfg& cfg, cudaStream_t stream);
int tcgen05_grid(size_t nbytes, const LaunchCfg& cfg);

}  // namespace tcr
