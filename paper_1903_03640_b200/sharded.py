"""Multi-GPU sharded reduction: the paper's two-level distributed reduction
(§II: "(1) local reduction and (2) distributed reduction ... the results
of different compute nodes must be merged with message passing"), B200-style:
one process per GPU, the local reduction is ``tcr_reduce_sum_f64`` on the
rank's contiguous shard, and the merge is ONE NCCL allreduce of the 8-byte
fp64 partials over NVLink/NVSwitch, followed by one rounding to binary32 on
the device (``tcr_round_f64_to_f32``).  Allreducing fp64 partials keeps the
cross-GPU combine from adding binary32 roundings to the error budget
(DESIGN.md §"Multi-GPU").

Segmented workloads shard by whole segments (element-count prefix on the
CSR offsets) and need no collective.

The reducer / finaliser are parameters so the host logic can be exercised
with the gloo backend on CPU (tests/test_multigpu_gloo.py); their defaults
are the library's CUDA entry points.
"""
from __future__ import annotations

import bisect


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced element range [lo, hi) of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return n_total * rank // world, n_total * (rank + 1) // world


def segment_shard(offsets, world: int, rank: int) -> tuple[int, int]:
    """Segments [j0, j1) owned by `rank`: whole segments, split where the
    element prefix crosses rank * total / world (no segment is cut)."""
    S = len(offsets) - 1
    if S < 0:
        raise ValueError("offsets must have num_segments + 1 entries")
    base, total = int(offsets[0]), int(offsets[-1]) - int(offsets[0])

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return S
        target = base + total * r // world
        return min(S, bisect.bisect_left(offsets, target, 0, S + 1))

    return cut(rank), cut(rank + 1)


def sharded_reduce_sum(x_local, out32, partial64, group=None, stream=None, reducer=None,
                       finalize=None):
    """Reduce this rank's shard, allreduce the fp64 partials, round once.

    x_local: this rank's shard (device fp16 tensor); out32: float32[1] result
    (replicated on every rank, like D' in Eq. 12); partial64: float64[1]
    scratch.  Stream-ordered; no host synchronisation.
    """
    import torch
    import torch.distributed as dist

    if reducer is None or finalize is None:
        import paper_1903_03640_b200 as tcr

        reducer = reducer or (lambda x, p, s: tcr.tcr_reduce_sum_f64(x, p, stream=s))
        finalize = finalize or (lambda p, o, s: tcr.tcr_round_f64_to_f32(p, o, stream=s))
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        reducer(x_local, partial64, stream)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(partial64, op=dist.ReduceOp.SUM, group=group)
        finalize(partial64, out32, stream)
    return out32


def sharded_reduce_sum_exact(x_local, out32, acc, group=None, stream=None, reducer=None,
                             finalize=None, dtype=None):
    """Exact sharded sum (NEXT-3): per-rank tcr_reduce_sum_exact_ex into the
    int64 exact state ``acc`` -- TCR_EXACT_ACC_WORDS (6: integer limbs of the
    sum in the type's unit plus special-value counts) for binary16 / fp8,
    TCR_EXACT_BF16_ACC_WORDS (27: eight exponent windows of three limbs, plus
    counts) for bfloat16 -- ONE int64 SUM allreduce (exact: limbs stay far
    below 2^63 for any realistic rank count), tcr_exact_finalize_ex.  The
    result is bitwise identical for every number of GPUs.
    """
    import torch
    import torch.distributed as dist

    if reducer is None or finalize is None:
        import paper_1903_03640_b200 as tcr

        # any exact-capable type: acc holds TCR_EXACT_ACC_WORDS (binary16 / fp8)
        # or TCR_EXACT_BF16_ACC_WORDS (bfloat16) int64
        code = tcr._dtype_of(x_local, dtype)
        tcr._check_acc(acc, code, "sharded_reduce_sum_exact")
        reducer = reducer or (lambda x, a, s: tcr.tcr_reduce_sum_exact_ex(x, acc=a, dtype=code,
                                                                           stream=s))
        finalize = finalize or (lambda a, o, s: tcr.tcr_exact_finalize_ex(a, code, out_f32=o,
                                                                           stream=s))
    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        reducer(x_local, acc, stream)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
        finalize(acc, out32, stream)
    return out32


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
