"""World-size-2 (and 3) CPU tests of the sharded path's host logic with the
gloo backend: shard ranges, segment sharding, and the fp64-partial allreduce
combine, with the exact oracle standing in for the per-GPU local reduction."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1903_03640_b200.sharded import segment_shard, shard_range


def test_shard_ranges_partition_exactly():
    for n in (0, 1, 7, 1 << 20, (1 << 33) + 5):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_segment_shard_whole_segments():
    import tcr_inputs as gen

    off = gen.offsets_from_lengths(gen.loguniform_lengths(1, 10_000), start=17)
    for world in (1, 2, 3, 8):
        rs = [segment_shard(off, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == 10_000
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        loads = [int(off[b] - off[a]) for a, b in rs]
        assert max(loads) - min(loads) <= 2 * 65536 + 1  # balanced up to a segment or two


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    import oracle
    import tcr_inputs as gen
    from paper_1903_03640_b200.sharded import shard_range, sharded_reduce_sum

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n, world, rank)
    bits = gen.generate(gen.SEED_C4, lo, hi - lo, gen.UNIFORM_01)

    def reducer(x, p, s):  # stand-in for tcr_reduce_sum_f64 on this rank's GPU
        p.fill_(oracle.exact_sum_fp16(x).f64())

    def finalize(p, o, s):  # stand-in for tcr_round_f64_to_f32
        o.fill_(float(np.float32(p.item())))

    out = torch.empty(1, dtype=torch.float32)
    part = torch.empty(1, dtype=torch.float64)
    sharded_reduce_sum(bits, out, part, reducer=reducer, finalize=finalize)
    q.put((rank, float(out.item())))
    dist.destroy_process_group()


def _worker_exact(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    import oracle
    import tcr_inputs as gen
    from paper_1903_03640_b200.sharded import shard_range, sharded_reduce_sum_exact

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n, world, rank)
    bits = gen.generate(gen.SEED_C4, lo, hi - lo, gen.WIDE)

    def reducer(x, acc, s):  # stand-in for tcr_reduce_sum_exact: limbs of the exact shard sum
        es = oracle.exact_sum_fp16(x)
        t = es.T
        acc.copy_(torch.tensor([t & ((1 << 40) - 1), (t >> 40) & ((1 << 40) - 1), t >> 80,
                                es.n_nan, es.n_pinf, es.n_ninf], dtype=torch.int64))

    def finalize(acc, o, s):  # stand-in for tcr_exact_finalize (host decode + RNE)
        a = acc.tolist()
        t = a[0] + (a[1] << 40) + (a[2] << 80)
        o.fill_(oracle.round_to_f32(t * oracle.UNIT))
        q.put((rank, t, float(o.item())))

    out = torch.empty(1, dtype=torch.float32)
    acc = torch.empty(6, dtype=torch.int64)
    sharded_reduce_sum_exact(bits, out, acc, reducer=reducer, finalize=finalize)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exact_limb_allreduce(world):
    import oracle
    import tcr_inputs as gen

    n = 2_000_003
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_exact, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    es = oracle.exact_sum_fp16(gen.generate(gen.SEED_C4, 0, n, gen.WIDE))
    assert {t for _, t, _ in res} == {es.T}          # integer allreduce is exact
    assert {g for _, _, g in res} == {es.f32()}      # bitwise, every rank, every world size


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_fp64_partial_allreduce(world):
    import oracle
    import tcr_inputs as gen

    n = 3_000_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    es = oracle.exact_sum_fp16(gen.generate(gen.SEED_C4, 0, n, gen.UNIFORM_01))
    vals = set(res.values())
    assert len(vals) == 1  # replicated on every rank
    g = vals.pop()
    assert oracle.within_tolerance(g, es)
    # fp64 partials of exact shard sums: the combine adds at most one fp64
    # rounding per rank, so the result is the correctly rounded fp32 here
    assert g == es.f32()
