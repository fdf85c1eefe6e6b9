/*
 * tcr.h -- C ABI of libtcr: tensor-core (MMA-encoded) fp16 sum reduction on
 * NVIDIA B200 (sm_100a).  From-scratch implementation of the hot path of
 * arXiv 1903.03640, "Analyzing GPU Tensor Core Potential for Fast
 * Reductions" (Carrasco, Vega, Navarro).
 *
 * Citations: "P:L" = line L of the paper text; section/equation
 * numbers follow the paper's LaTeX auto-numbering.
 *
 * The operation (§III Eq. 2):  R(X) = sum_{i=1..n} x_i,
 * with x_i IEEE-754 binary16.  The library encodes it as the paper does
 * (§IV.A, Eq. 9-14): each 16x16 tile A of 256 inputs is
 * multiplied by an all-ones matrix, D = A x 1 + C, which puts the tile's
 * row sums in every column (Eq. 10); the accumulator C is carried
 * across a bounded chain of tiles; a second MMA with the ones in the A
 * position, D' = 1 x D (Eq. 11-12), collapses row sums to one
 * scalar replicated in every entry; and the level recursion R_tc
 * (Eq. 13-14) continues across warps, CTAs and the grid inside
 * ONE launch (the inter-level barrier, which the paper gets from kernel
 * termination, is a last-CTA completion ticket).
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - x, offsets and out are DEVICE pointers (cudaMalloc / torch tensors)
 *    owned by the caller, except in tcr_reduce_sum_host.  They must stay
 *    valid until the enqueued work completes; the library never frees them.
 *  - x holds binary16 bit patterns (tcr_half), 2-byte aligned; any 16-byte
 *    misalignment is handled internally.  out must be 4-byte aligned
 *    (8-byte for double).
 *  - stream: a cudaStream_t (tcr_stream is layout-identical), NULL = the
 *    legacy default stream.  Every call is stream-ordered and asynchronous
 *    (no host synchronisation) except tcr_reduce_sum_host.
 *  - Accuracy contract (north star, BASELINE.json): for finite inputs the
 *    binary32 result g satisfies |g - R(X)| <= 2^-20 * sum |x_i|.  The
 *    paper leaves the precision of the tensor-core reduction open;
 *    this bound is the library's, not the paper's.  NaN/inf inputs
 *    propagate as IEEE addition would.
 *  - Results are bitwise deterministic for a given (device, n, x, algo,
 *    configuration, library build): the order of every floating-point
 *    operation is fixed, no floating-point atomics are used.
 *  - n == 0 (or an empty segment) yields +0.0.
 *  - Errors: a status is returned, nothing is thrown across the ABI.
 *    TCR_ERR_INVALID_VALUE for NULL pointers with n > 0, misaligned
 *    pointers, or an unknown algo/config key; TCR_ERR_UNSUPPORTED_DEVICE if
 *    the current device is not compute capability 10.x (there is no
 *    fallback of any kind); TCR_ERR_OUT_OF_MEMORY if the workspace cannot be
 *    allocated; TCR_ERR_CUDA for a CUDA error (text in tcr_last_error()).
 *    Asynchronous device faults surface at the caller's next synchronisation.
 *  - Workspace: the library owns a small per-(device, stream) workspace
 *    (fp64 partials of the CTAs, a completion ticket, scheduler counters),
 *    allocated on the first call for that stream and reused.  The first
 *    call on a stream must therefore not be made while that stream is being
 *    captured into a CUDA graph.  tcr_release_workspaces() frees them.
 *  - Threading: calls are reentrant; concurrent calls on distinct streams
 *    are safe (separate workspaces); calls on one stream are serialised by
 *    stream order.
 */
#ifndef TCR_H_
#define TCR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCR_VERSION 100 /* 1.0.0 */

typedef uint16_t tcr_half;              /* IEEE-754 binary16 bit pattern */
typedef struct CUstream_st *tcr_stream; /* == cudaStream_t / CUstream     */

typedef enum {
    TCR_OK = 0,
    TCR_ERR_INVALID_VALUE = 1,
    TCR_ERR_UNSUPPORTED_DEVICE = 2,
    TCR_ERR_OUT_OF_MEMORY = 3,
    TCR_ERR_CUDA = 4
} tcr_status;

/* Kernel selection for tcr_reduce_sum_algo / the _config default. */
typedef enum {
    TCR_ALGO_DEFAULT = 0, /* TCR_CFG_DEFAULT_ALGO; its default, 0 = auto by
                             size: tcgen05 (dynamic tail) for binary16 / fp8
                             from 512 MiB of input, mma.sync below and for
                             bfloat16 -- see tcr_default_algo              */
    TCR_ALGO_MMA_SYNC = 1, /* mma.sync m16n8k16 (A from 128-bit loads)       */
    TCR_ALGO_TCGEN05 = 2, /* cp.async.bulk -> SMEM -> tcgen05.mma, D in TMEM */
    TCR_ALGO_SHUFFLE = 3, /* classic comparison path (§II): fp32
                             FADD chains + shfl_xor tree, no tensor cores    */
    TCR_ALGO_BULK_MMA = 4 /* cp.async.bulk (TMA) -> SMEM ring -> ld.shared.v4 ->
                             mma.sync m16n8k16 by 8 consumer warps           */
} tcr_algo;

/* Input element type for the _ex entry points (NEXT-4). */
typedef enum {
    TCR_DTYPE_F16 = 0,  /* IEEE-754 binary16 (the north star)                */
    TCR_DTYPE_BF16 = 1, /* bfloat16: the same MMA encoding with .bf16 / kind::f16-BF16
                           operands and B = bfloat16 ones                    */
    TCR_DTYPE_E4M3 = 2, /* OCP fp8 E4M3FN (1 byte): mma.sync (the default): each
                           512-element tile is converted exactly to binary16 and
                           reduced as two m16n8k16 against binary16 ones (what
                           sm_100a runs for m16n8k32 .e4m3); or tcgen05
                           kind::f8f6f4 with B = fp8 ones */
    TCR_DTYPE_E5M2 = 3  /* OCP fp8 E5M2 (1 byte), as E4M3                     */
} tcr_dtype;

/*
 * tcr_reduce_sum -- R(X) of n binary16 values x[0..n) into *out (binary32).
 * The north-star entry point: MMA-encoded, one kernel launch, writes *out
 * on the device.  (Eq. 2; method P:169-236 Eq. 9-14.)
 */
tcr_status tcr_reduce_sum(const tcr_half *x, size_t n, float *out, tcr_stream stream);

/*
 * tcr_reduce_sum_shuffle -- same contract as tcr_reduce_sum, computed by the
 * classic warp-shuffle tree reduction (the paper's comparison algorithm,
 * P:83-85 and P:113-137) instead of MMAs.
 */
tcr_status tcr_reduce_sum_shuffle(const tcr_half *x, size_t n, float *out, tcr_stream stream);

/*
 * tcr_reduce_sum_f64 -- same reduction as tcr_reduce_sum, but writes the
 * binary64 total *before* the final rounding to binary32.  Used as the
 * per-GPU partial of a sharded reduction (the paper's "local reduction"
 * of a distributed reduction), so the cross-GPU combine does not add
 * binary32 roundings.
 */
tcr_status tcr_reduce_sum_f64(const tcr_half *x, size_t n, double *out, tcr_stream stream);

/*
 * tcr_reduce_sum_algo -- explicit kernel choice.  Writes the binary32
 * result to out_f32 and/or the binary64 total to out_f64 (either may be
 * NULL, not both).
 */
tcr_status tcr_reduce_sum_algo(const tcr_half *x, size_t n, float *out_f32, double *out_f64,
                               tcr_algo algo, tcr_stream stream);

/*
 * tcr_reduce_sum_ex -- tcr_reduce_sum_algo for any supported input type:
 * x holds n elements of `dtype` (binary16 / bfloat16 / fp8 bit patterns;
 * element-aligned; fp8 elements are 1 byte).
 * Same accuracy contract (|g - R| <= 2^-20 * sum|x_i| while the sum is
 * inside the binary32 range) and error behaviour; TCR_ERR_INVALID_VALUE for
 * an unknown dtype.  (Other entry points taking a dtype:
 * tcr_reduce_sum_segmented_ex, tcr_reduce_sum_batched_ex,
 * tcr_reduce_sum_host_ex, tcr_reduce_sum_exact_ex, tcr_reduce_sum_peer.)
 */
tcr_status tcr_reduce_sum_ex(const void *x, size_t n, tcr_dtype dtype, float *out_f32,
                             double *out_f64, tcr_algo algo, tcr_stream stream);

/*
 * tcr_reduce_sum_segmented -- per-segment R over CSR offsets:
 * out[j] = R(x[offsets[j] .. offsets[j+1])) for j in [0, num_segments).
 * offsets: device int64[num_segments + 1], non-decreasing, offsets[0] >= 0,
 * all within the caller's x buffer (not checked on the device).  out:
 * device float[num_segments].  Each segment is reduced by the MMA encoding
 * with its unaligned head and tail zero-masked (the paper's zero padding of
 * the trailing group, reading G5).  out[j] corresponds exactly to segment j.
 * Segments may be read as whole aligned 16-byte vectors, i.e. up to 14 bytes
 * outside [offsets[0], offsets[S]) but never outside the 16-byte-aligned
 * chunks that contain segment data.
 */
tcr_status tcr_reduce_sum_segmented(const tcr_half *x, const int64_t *offsets,
                                    size_t num_segments, float *out, tcr_stream stream);
tcr_status tcr_reduce_sum_segmented_shuffle(const tcr_half *x, const int64_t *offsets,
                                            size_t num_segments, float *out, tcr_stream stream);
/* Segmented for any input type (binary16, bfloat16, fp8 E4M3 / E5M2; offsets
 * in elements of that type); algo = DEFAULT / MMA_SYNC (MMA) or SHUFFLE. */
tcr_status tcr_reduce_sum_segmented_ex(const void *x, tcr_dtype dtype, const int64_t *offsets,
                                       size_t num_segments, float *out, tcr_algo algo,
                                       tcr_stream stream);

/*
 * tcr_reduce_sum_batched -- num_segments contiguous segments of segment_len
 * elements each: out[j] = R(x[j*segment_len .. (j+1)*segment_len)).
 * Same accuracy contract per segment as tcr_reduce_sum; bitwise
 * deterministic.  Kernel choice (internal, TCR_CFG_ROWS_TC05): rows of any
 * format with x 16-byte aligned, a row pitch that is a multiple of 16 bytes
 * and at most 6144 bytes (not binary16 / bfloat16 segment_len 1024) and at
 * least 256 x SMs segments run on tcgen05 with 256 segments per TMA tensor
 * box, each segment a row of A (Eq. 9-10);
 * otherwise the mma.sync kernels (16 segments as the 16 rows of A for
 * segment_len % 32 == 0 up to 2048, whole-tile rows, or the union stream).
 */
tcr_status tcr_reduce_sum_batched(const tcr_half *x, size_t num_segments, size_t segment_len,
                                  float *out, tcr_stream stream);
tcr_status tcr_reduce_sum_batched_shuffle(const tcr_half *x, size_t num_segments,
                                          size_t segment_len, float *out, tcr_stream stream);
/* Batched for any input type (segment_len in elements of that type). */
tcr_status tcr_reduce_sum_batched_ex(const void *x, tcr_dtype dtype, size_t num_segments,
                                     size_t segment_len, float *out, tcr_algo algo,
                                     tcr_stream stream);

/*
 * tcr_reduce_sum_host -- end-to-end form: x is a HOST pointer (pinned
 * memory for full PCIe bandwidth; pageable works), *out is a HOST float.
 * The library streams x to the device in chunks through its own staging
 * buffers on `stream`, reduces each chunk with the default MMA kernel into
 * a binary64 partial, combines the partials in chunk order on the device,
 * copies the binary32 result back and synchronises `stream` before
 * returning.  Same accuracy contract as tcr_reduce_sum.
 */
tcr_status tcr_reduce_sum_host(const tcr_half *x, size_t n, float *out, tcr_stream stream);
/* The same for any input type (chunks of 128 MiB of input bytes). */
tcr_status tcr_reduce_sum_host_ex(const void *x, size_t n, tcr_dtype dtype, float *out,
                                  tcr_stream stream);

/*
 * tcr_reduce_sum_exact -- NEXT-3: the EXACT sum (no rounding before the
 * final conversion).  Each binary16 is placed bit-exactly into a scaled
 * binary64 (x * 2^-1008, subnormals included); <= 1024 of them are added
 * exactly per accumulator, flushed into 128-bit integers in units of 2^-24,
 * and combined exactly across warps, CTAs and the grid (one launch).
 * Outputs (each may be NULL, not all):
 *   acc[6]  (device int64): {l0, l1, l2, n_nan, n_pinf, n_ninf} with the
 *           exact sum T = (l0 + l1*2^40 + l2*2^80) * 2^-24, l0, l1 in
 *           [0, 2^40).  Integer-summing acc[] of several shards (e.g. an
 *           NCCL int64 SUM allreduce) is exact; see tcr_exact_finalize.
 *   out_f32 / out_f64: the correctly rounded (RNE) value of T, or the IEEE
 *           special value if any input was NaN / inf.
 * Bitwise identical to the exact oracle for every input; independent of
 * grid size, thread count and (for sharded use) the number of GPUs.
 */
tcr_status tcr_reduce_sum_exact(const tcr_half *x, size_t n, int64_t *acc, float *out_f32,
                                double *out_f64, tcr_stream stream);

/*
 * tcr_reduce_sum_exact_ex -- tcr_reduce_sum_exact for every input type:
 *   binary16, fp8 E4M3 / E5M2 (every fp8 value is a binary16 value, converted
 *   exactly on the fly): the same acc[6] state in units of 2^-24, the same
 *   tcr_exact_finalize;
 *   bfloat16 (range 2^-133..2^128): eight 32-exponent windows, each summed
 *   exactly (binary64 fast path for iterations inside one window, integer
 *   slow path otherwise), assembled in a 384-bit integer and rounded once;
 *   acc (if not NULL) holds TCR_EXACT_BF16_ACC_WORDS int64: per window k
 *   three limbs (I_k = a[3k] + a[3k+1] 2^40 + a[3k+2] 2^80, in units of
 *   2^-133 for k = 0 and 2^(32k-134) above), then n_nan, n_pinf, n_ninf --
 *   integer-summable across GPUs like the binary16 limbs.
 * acc length: the ABI takes a bare pointer, so the CALLER must provide at
 * least TCR_EXACT_ACC_WORDS int64 for binary16 / fp8 and
 * TCR_EXACT_BF16_ACC_WORDS for bfloat16 (a shorter buffer is overrun; the
 * Python binding checks the length).  tcr_exact_finalize_ex must be called
 * with the same dtype as the reduction that wrote acc.
 * Bitwise equal to the exact oracle of the type.
 * Kernels (TCR_CFG_EXACT_BULK): binary16 from 128 MiB on the TMA-fed exact
 * kernel; fp8 E4M3 from 64 MiB on the tcgen05 reduction itself (its rows of
 * 64 E4M3 values are exact in binary32, the combine is integer), followed,
 * when acc is given, by a second kernel that counts NaN bytes only if a NaN
 * went by -- so this entry may enqueue two kernels.
 */
#define TCR_EXACT_ACC_WORDS 6
#define TCR_EXACT_BF16_ACC_WORDS 27
tcr_status tcr_reduce_sum_exact_ex(const void *x, size_t n, tcr_dtype dtype, int64_t *acc,
                                   float *out_f32, double *out_f64, tcr_stream stream);

/* tcr_exact_finalize -- RNE binary32 / binary64 of an (allreduced) acc[6]. */
/* tcr_exact_finalize_ex -- the same for an acc of any exact-capable dtype
 * (6 words for binary16 / fp8, 27 for bfloat16). */
tcr_status tcr_exact_finalize_ex(const int64_t *acc, tcr_dtype dtype, float *out_f32,
                                 double *out_f64, tcr_stream stream);
tcr_status tcr_exact_finalize(const int64_t *acc, float *out_f32, double *out_f64,
                              tcr_stream stream);

/*
 * tcr_round_f64_to_f32 -- out[0] = (float)in[0], round-to-nearest-even, on
 * the device (finaliser of a sharded reduction after the allreduce of the
 * binary64 partials).
 */
tcr_status tcr_round_f64_to_f32(const double *in, float *out, tcr_stream stream);

/*
 * ---------------------------------------------------------------------------
 * Fused cross-GPU combine (NEXT-2; the paper's distributed reduction, P:89,
 * §II: "the results of different compute nodes must be merged with message
 * passing").  Instead of a separate NCCL allreduce, the kernel's last CTA
 * pushes the rank's fp64 partial over NVLink into every peer's MAILBOX
 * (a TCR_PEER_MAILBOX_BYTES device allocation per rank, mapped into the
 * other processes by CUDA IPC), waits for the peers' partials in its own
 * mailbox, sums them in rank order 0..P-1 and writes the group total: every
 * rank gets the bitwise identical result (D' replicated, Eq. 12) from ONE
 * launch, with no host synchronisation.  Each mailbox counts its rank's
 * combines on the device (the epoch that tags the partials), so the launch
 * can be captured in a CUDA graph and replayed.  A mailbox therefore belongs
 * to ONE group: every rank of the group must have made the same number of
 * combines on it (using a mailbox in two groups, e.g. alone and then in a
 * group of 8, desynchronises the epochs and the waits run into
 * TCR_CFG_PEER_TIMEOUT_MS, returning NaN with the error word set).
 *
 * Group setup (once): each rank tcr_peer_mailbox_alloc()s its mailbox,
 * exports it with tcr_peer_ipc_handle(), the handles are exchanged out of
 * band (e.g. torch.distributed.all_gather_object), and each rank
 * tcr_peer_ipc_open()s the peers' handles.  mailboxes[r] is then rank r's
 * mailbox as seen by this process (its own pointer for r == rank).
 * Teardown: all ranks quiesce (stream sync + a barrier), close the peers'
 * mappings (tcr_peer_ipc_close), then free their own mailbox.
 * ---------------------------------------------------------------------------
 */
#define TCR_MAX_PEERS 8           /* ranks per peer group (one NVLink node) */
#define TCR_PEER_MAILBOX_BYTES 2048
#define TCR_IPC_HANDLE_BYTES 64

/* Allocates (cudaMalloc, IPC-exportable) and zeroes a mailbox on the current
 * device; synchronous.  Free with tcr_peer_mailbox_free. */
tcr_status tcr_peer_mailbox_alloc(void **mailbox);
tcr_status tcr_peer_mailbox_free(void *mailbox);
/* Stream-ordered zeroing: clears the error word and restarts the combine
 * count; every rank of the group must reset before the next combine. */
tcr_status tcr_peer_mailbox_reset(void *mailbox, tcr_stream stream);
/* Synchronous read of the mailbox's error word: *timed_out = 1 if a combine
 * on this rank gave up waiting (its result was NaN); reset to clear. */
tcr_status tcr_peer_mailbox_error(const void *mailbox, int *timed_out);
/* handle: host buffer of TCR_IPC_HANDLE_BYTES (cudaIpcMemHandle_t). */
tcr_status tcr_peer_ipc_handle(const void *mailbox, void *handle);
tcr_status tcr_peer_ipc_open(const void *handle, void **peer_mailbox);
tcr_status tcr_peer_ipc_close(void *peer_mailbox);

/*
 * tcr_reduce_sum_peer -- sum of this rank's shard x[0..n) (dtype as in
 * tcr_reduce_sum_ex) fused with the group combine: out_f32[0] / out_f64[0]
 * = the total over all nranks shards (binary64 sum of the ranks' fp64
 * partials in rank order; out_f32 its RNE rounding).  One kernel launch on
 * `stream`.
 *   algo:      TCR_ALGO_DEFAULT (as tcr_reduce_sum, resolved for the per-rank
 *              shard size), MMA_SYNC, TCGEN05 (r02: the combine fused into the
 *              tcgen05 kernel's last CTA) or SHUFFLE.
 *   mailboxes: HOST array of nranks device pointers, indexed by rank.
 *   nranks:    1..TCR_MAX_PEERS; rank: this process's index.
 * Every rank of the group must make the same sequence of calls, each rank's
 * calls stream-ordered (one stream, or ordered by events); a rank whose peers do
 * not arrive within TCR_CFG_PEER_TIMEOUT_MS writes NaN and sets its
 * mailbox's error word (the group must then be reset on every rank).
 */
tcr_status tcr_reduce_sum_peer(const void *x, size_t n, tcr_dtype dtype, tcr_algo algo,
                               void *const *mailboxes, int nranks, int rank, float *out_f32,
                               double *out_f64, tcr_stream stream);

/*
 * tcr_reduce_sum_peer_emulated -- the same kernel and protocol with all
 * nranks ranks emulated in ONE cooperative launch on this device (grid slice
 * r = rank r, reducing the shard [r*n/P, (r+1)*n/P) of x, as
 * shard_range() in sharded.py): testing and measurement of the fused
 * combine on a single GPU.  out_f32 / out_f64: device arrays of nranks
 * entries (rank r's result in [r]); mailboxes as above (nranks distinct
 * mailboxes, any of which may be IPC mappings).
 */
tcr_status tcr_reduce_sum_peer_emulated(const void *x, size_t n, tcr_dtype dtype, tcr_algo algo,
                                        void *const *mailboxes, int nranks, float *out_f32,
                                        double *out_f64, tcr_stream stream);

/*
 * tcr_reduce_sum_exact_peer -- tcr_reduce_sum_exact of this rank's binary16
 * shard fused with the group combine of the int64 limb states (NEXT-2 x
 * NEXT-3): acc[0..6) (may be NULL) receives the group's summed limbs and
 * out_f32 / out_f64 their correctly rounded value -- bitwise identical on
 * every rank and for every number of ranks.  Same mailboxes, epochs, stream
 * ordering and timeout behaviour as tcr_reduce_sum_peer (both kinds of
 * combine may be interleaved on one group; each advances its epoch).
 * binary16 ONLY: x is decoded as binary16 (a bfloat16 or fp8 buffer would be
 * misread, an fp8 one over-read by 2x); for other types use
 * tcr_reduce_sum_exact_ex + an int64 allreduce of its state.
 */
tcr_status tcr_reduce_sum_exact_peer(const tcr_half *x, size_t n, void *const *mailboxes,
                                     int nranks, int rank, int64_t *acc, float *out_f32,
                                     double *out_f64, tcr_stream stream);
/* All ranks emulated in one cooperative launch (acc: 6 words per rank,
 * out_f32 / out_f64: one per rank), as tcr_reduce_sum_peer_emulated. */
tcr_status tcr_reduce_sum_exact_peer_emulated(const tcr_half *x, size_t n,
                                              void *const *mailboxes, int nranks, int64_t *acc,
                                              float *out_f32, double *out_f64, tcr_stream stream);

/*
 * tcr_probe_mma -- hardware characterisation (not part of the reduction):
 * executes ONE MMA of the given algo (TCR_ALGO_MMA_SYNC: m16n8k16;
 * TCR_ALGO_TCGEN05: M=128,N=16,K=16) with A = a (row-major 16x16 for
 * mma.sync / 128x16 for tcgen05, binary16), B = all ones and C = c
 * (binary32, one value per row of A), and writes D's first column to d.
 * a: device tcr_half[16*16] or [128*16]; c, d: device float[16] or [128].
 * Used by the tests to record whether the tensor-core fp32 accumulate
 * rounds to nearest or truncates (reading G10).
 */
tcr_status tcr_probe_mma(const tcr_half *a, const float *c, float *d, tcr_algo algo,
                         tcr_stream stream);

/*
 * tcr_reduce_sum_paper_f16 -- STUDY MODE (NEXT-1, not the product path): the
 * paper's algorithm taken literally (§IV.A, Eq. 9-14): per group
 * of 256 inputs D = A x 1 and D' = 1 x D with fp16 accumulation
 * (mma.sync .f16.f16.f16.f16), D'_{1,1} written to memory as binary16, and
 * one kernel launch per level until one value is left (ceil(log_256 n)
 * launches).  out: device float, the final binary16 value widened.  Exposes
 * the fp16 precision loss the paper leaves open -- overflow to inf
 * once a partial exceeds 65504 -- and the cost of the per-level relaunch that
 * the product path replaces with one launch.  Library-owned scratch of
 * ~n/255 binary16 per stream (grown on demand).
 */
tcr_status tcr_reduce_sum_paper_f16(const tcr_half *x, size_t n, float *out, tcr_stream stream);

/*
 * tcr_reduce_sum_study_fp32 -- STUDY MODE (NEXT-1 comparison point, not the
 * product path): the classic reduction entirely in binary32 -- the shuffle
 * path's loads and tree with no fp64 anywhere -- naive (kahan = 0) or with
 * Kahan compensation of the per-lane and grid-level sums (kahan = 1).
 */
tcr_status tcr_reduce_sum_study_fp32(const tcr_half *x, size_t n, int kahan, float *out,
                                     tcr_stream stream);

/*
 * tcr_probe_collapse -- the level-2 collapse D' = 1 x D (Eq. 11-12) in
 * isolation: lane l of one warp holds in[l] (device double[32]); out[l]
 * (device double[32]) receives lane l's result of the collapse used by the
 * kernels (TCR_ALGO_MMA_SYNC: three m8n8k4 f64 DMMAs with ones in A;
 * TCR_ALGO_SHUFFLE: the shfl_xor tree).  Every lane gets the sum (the
 * replication of Eq. 12).  For the tests (SURVEY T-D(iii)).
 */
tcr_status tcr_probe_collapse(const double *in, double *out, tcr_algo algo, tcr_stream stream);

/* Tuning knobs (process-wide; defaults are the measured best on B200). */
typedef enum {
    TCR_CFG_DEFAULT_ALGO = 0,     /* tcr_algo used by tcr_reduce_sum; 0 (the
                                   * default) = auto by input size: tcgen05 for
                                   * binary16 / fp8 from 512 MiB, mma.sync below
                                   * and for bfloat16          */
    TCR_CFG_BLOCKS_PER_SM = 1,    /* CTAs per SM of the streaming kernels   */
    TCR_CFG_UNROLL = 2,           /* 16-byte loads in flight per lane (mma.sync/shuffle):
                                     4, 8, 16, or 0 = auto (default: 16 below
                                     2^26 elements, 4 from there on)            */
    TCR_CFG_TC05_STAGES = 3,      /* SMEM ring stages of the tcgen05 kernel */
    TCR_CFG_TC05_STAGE_KB = 4,    /* KiB per stage of the tcgen05 kernel    */
    TCR_CFG_CHAIN = 5,            /* mma_sync/shuffle: carried chain K, tiles per
                                     fp32 accumulator before its fp64 flush
                                     (rounded to a multiple of unroll/2; at
                                     unroll 16 at least 4)                     */
    TCR_CFG_TC05_SLOTS = 6,       /* tcgen05: independent TMEM accumulators per
                                     buffer (1, 2, 4, 8, 16)                    */
    TCR_CFG_TC05_CHAIN = 7,       /* tcgen05: MMAs carried per accumulator (K) */
    TCR_CFG_TC05_CTAS_PER_SM = 8, /* tcgen05: CTAs per SM (1..4); 0 (default) =
                                   * auto: 1 from 256 MiB of input, else 3 with
                                   * <= 2 stages each                          */
    TCR_CFG_TC05_PREFETCH = 9,    /* tcgen05: L2 prefetch distance in chunks (0 = off) */
    TCR_CFG_TC05_SPLIT = 10,      /* tcgen05: bulk copies per stage (1, 2, 4, 8) */
    TCR_CFG_TC05_INTERLEAVE = 11, /* tcgen05: 0 = each CTA streams a contiguous run
                                     of chunks, 1 = chunks dealt round-robin    */
    TCR_CFG_EXACT_UNROLL = 12,    /* exact kernel: 16-byte loads per lane in flight (4, 8) */
    TCR_CFG_EXACT_BLOCKS_PER_SM = 13, /* exact kernel: CTAs per SM (1..8)       */
    TCR_CFG_BULK_STAGES = 14,     /* bulk kernel: SMEM ring stages (2..32)      */
    TCR_CFG_BULK_STAGE_KB = 15,   /* bulk kernel: KiB per stage (4..64, x4)     */
    TCR_CFG_BULK_CTAS_PER_SM = 16, /* bulk kernel: CTAs per SM (clamped by SMEM) */
    TCR_CFG_PEER_TIMEOUT_MS = 17,  /* fused peer combine: bound on the wait for the
                                     peers' partials (default 10000 ms)          */
    TCR_CFG_PDL = 18,             /* 1 (default): the reduction kernels (streaming,
                                   * tcgen05, bulk, exact, segmented / batched) are
                                   * launched with programmatic dependent launch -- a
                                   * call's CTAs are scheduled while the previous kernel
                                   * on the stream drains and wait (griddepcontrol.wait)
                                   * for its completion before touching global memory;
                                   * results are bitwise identical either way (the fused
                                   * peer kernels always launch plainly); 0: plain launch */
    TCR_CFG_TC05_DYNAMIC = 19,    /* tcgen05: percent (0..100) of the chunks handed
                                   * out at run time from a chunk counter (the
                                   * dynamic tail: every CTA first streams its own
                                   * contiguous run, then takes the remaining chunks
                                   * one at a time) -- 0 = static partition.  With a
                                   * nonzero value the rounds are combined exactly
                                   * (integer units of 2^-24), so the result does not
                                   * depend on which CTA took which chunk; binary16
                                   * and fp8 (bfloat16 always uses the static
                                   * partition; so do runs shorter than
                                   * TCR_CFG_TC05_DYN_MIN_RUN); default 8
                                   *                             */
    TCR_CFG_TC05_DYN_MIN_RUN = 20, /* tcgen05: the dynamic tail only when every CTA
                                   * streams at least this many chunks (default 32;
                                   * 0 = whenever TCR_CFG_TC05_DYNAMIC > 0)       */
    TCR_CFG_ROWS_TC05 = 21,       /* batched (MMA): 1 (default) = fixed-length rows
                                   * on tcgen05 where applicable -- any format,
                                   * x 16-byte aligned, row pitch a multiple of
                                   * 16 bytes up to 6144 (not 16-bit L = 1024),
                                   * at least 256 x SMs segments:
                                   * 128 segments are the 128 rows of A, loaded by
                                   * TMA tensor copies; 0 = the
                                   * mma.sync kernels                             */
    TCR_CFG_ROWS_TC05_STAGES = 22, /* that kernel's SMEM ring stages of 32 KiB
                                   * (2..6, default 4)                           */
    TCR_CFG_EXACT_BULK = 23       /* exact: 1 (default) = binary16 from 128 MiB on
                                   * the TMA-fed kernel with the dynamic tail, fp8
                                   * E4M3 from 64 MiB on the tcgen05 dynamic-tail
                                   * kernel (its rows are exact; + a NaN count)
                                   * (cp.async.bulk ring, 8 consumer warps, chunk
                                   * tickets per TCR_CFG_TC05_DYNAMIC; DESIGN.md
                                   * §18); 2 = that kernel at every size; 0 = the
                                   * LDG kernel at every size                     */
} tcr_config_key;
tcr_status tcr_set_config(tcr_config_key key, int value);
int tcr_get_config(tcr_config_key key); /* -1 for an unknown key */

const char *tcr_status_string(tcr_status s);
const char *tcr_last_error(void);        /* thread-local detail of the last error */
tcr_status tcr_release_workspaces(void); /* caller guarantees no in-flight work   */
uint64_t tcr_launch_count(void);         /* kernels launched by this library so far */
/* The kernel TCR_ALGO_DEFAULT resolves to for n elements of `dtype` under the
 * current configuration (never TCR_ALGO_DEFAULT); no device work. */
tcr_algo tcr_default_algo(size_t n, tcr_dtype dtype);
int tcr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TCR_H_ */
