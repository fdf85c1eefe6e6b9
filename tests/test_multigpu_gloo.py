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


# ---------------------------------------------------------------------------
# NEXT-2 fused peer combine: PeerGroup's host logic (mailbox allocation, IPC
# handle exchange over the process group, rank-indexed mailbox table, epoch
# counting, teardown order) under gloo, with a CPU stand-in for the device
# side.  The stand-in implements the mailbox protocol of tcr_peer.cuh on
# shared memory between the rank processes (value, then flag = epoch, into
# slot [epoch & 1][rank] of every rank's mailbox; wait for all flags of the
# own mailbox; rank-ordered sum), so many epochs with random skew between
# ranks also exercise the two-parity reuse argument of tcr_peer.cuh.
# ---------------------------------------------------------------------------


class _ShmPeerLib:
    TCR_MAX_PEERS = 8

    def __init__(self, tag, rank):
        self.tag, self.rank, self.shm, self.calls = tag, rank, {}, []

    def _buf(self, p):
        return self.shm[p].buf

    def tcr_peer_mailbox_alloc(self):
        from multiprocessing import shared_memory

        s = shared_memory.SharedMemory(name=f"tcr{self.tag}r{self.rank}", create=True, size=512)
        s.buf[:512] = bytes(512)
        self.shm[1000 + self.rank] = s
        self.calls.append(("alloc",))
        return 1000 + self.rank

    def tcr_peer_ipc_handle(self, mbox):
        return self.shm[mbox].name.encode().ljust(64, b"\0")

    def tcr_peer_ipc_open(self, handle):
        from multiprocessing import shared_memory

        name = handle.rstrip(b"\0").decode()
        s = shared_memory.SharedMemory(name=name)
        p = 2000 + int(name.rsplit("r", 1)[1])
        self.shm[p] = s
        self.calls.append(("open", p))
        return p

    def tcr_peer_ipc_close(self, p):
        self.calls.append(("close", p))
        self.shm.pop(p).close()

    def tcr_peer_mailbox_free(self, p):
        self.calls.append(("free", p))
        s = self.shm.pop(p)
        s.close()
        s.unlink()

    def tcr_peer_mailbox_error(self, p):
        return False

    def tcr_reduce_sum_peer(self, x, mailboxes, rank, out_f32=None, out_f64=None,
                            algo=None, stream=None):
        import struct
        import time

        import oracle

        v = oracle.exact_sum_fp16(x).f64()  # stand-in for the rank's fp64 partial
        own = self._buf(mailboxes[rank])
        epoch = struct.unpack("<Q", bytes(own[264:272]))[0] + 1  # device-side combine counter
        P, par = len(mailboxes), epoch & 1
        off = lambda src: (par * 8 + src) * 16
        for d in range(P):  # push to every peer: value, then flag
            if d == rank:
                continue
            b = self._buf(mailboxes[d])
            b[off(rank) + 8:off(rank) + 16] = struct.pack("<d", v)
            b[off(rank):off(rank) + 8] = struct.pack("<Q", epoch)
        got = []
        for r in range(P):  # wait in the own mailbox (own partial: no round trip)
            if r == rank:
                got.append(v)
                continue
            t0 = time.time()
            while struct.unpack("<Q", bytes(own[off(r):off(r) + 8]))[0] != epoch:
                assert time.time() - t0 < 60, "peer never arrived"
                time.sleep(0.0005)
            got.append(struct.unpack("<d", bytes(own[off(r) + 8:off(r) + 16]))[0])
        own[264:272] = struct.pack("<Q", epoch)
        tot = 0.0
        for g in got:  # rank order
            tot += g
        self.calls.append(("reduce", tuple(mailboxes), rank, epoch))
        out_f64.fill_(tot)


def _worker_peer(rank, world, port, tag, epochs, q):
    import random
    import time

    import torch
    import torch.distributed as dist

    import tcr_inputs as gen
    from paper_1903_03640_b200.peer import PeerGroup
    from paper_1903_03640_b200.sharded import shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _ShmPeerLib(tag, rank)
    grp = PeerGroup(lib=lib)
    assert grp.mailboxes[rank] == grp.mailbox
    assert sorted(grp.mailboxes) == sorted([1000 + rank] + [2000 + r for r in range(world) if r != rank])
    assert all(grp.mailboxes[r] == 2000 + r for r in range(world) if r != rank)
    rng = random.Random(rank * 7919 + 1)
    res = []
    out = torch.empty(1, dtype=torch.float64)
    n = 50_001
    for e in range(epochs):
        time.sleep(rng.random() * 0.004)  # skew between ranks
        lo, hi = shard_range(n, world, rank)
        grp.reduce_sum(gen.generate(100 + e, lo, hi - lo, gen.UNIFORM_PM1), out_f64=out)
        res.append(float(out.item()))
    assert grp.calls == epochs
    grp.close()
    kinds = [c[0] for c in lib.calls]
    assert kinds[0] == "alloc" and kinds[-1] == "free"
    assert kinds.index("free") > max(i for i, k in enumerate(kinds) if k == "close")
    assert [c[3] for c in lib.calls if c[0] == "reduce"] == list(range(1, epochs + 1))
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_gloo_peer_group_protocol(world):
    import oracle
    import tcr_inputs as gen
    from paper_1903_03640_b200.sharded import shard_range

    epochs, n = 40, 50_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"{os.getpid()}x{port}"
    ps = [ctx.Process(target=_worker_peer, args=(r, world, port, tag, epochs, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for e in range(epochs):
        parts = [oracle.exact_sum_fp16(gen.generate(100 + e, *(lambda a, b: (a, b - a))(
            *shard_range(n, world, r)), gen.UNIFORM_PM1)).f64() for r in range(world)]
        want = 0.0
        for v in parts:
            want += v
        assert {res[r][e] for r in range(world)} == {want}, e  # replicated, rank-ordered


class _FailingPeerLib(_ShmPeerLib):
    def tcr_peer_mailbox_alloc(self):
        if self.rank == 1:
            raise RuntimeError("simulated allocation failure")
        return super().tcr_peer_mailbox_alloc()


def _worker_peer_fail(rank, world, port, tag, q):
    import torch.distributed as dist

    from paper_1903_03640_b200.peer import PeerGroup

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _FailingPeerLib(tag, rank)
    try:
        PeerGroup(lib=lib)
        q.put((rank, "constructed"))
    except RuntimeError as e:
        q.put((rank, "raised" if "rank(s) [1]" in str(e) else f"other: {e}"))
    dist.destroy_process_group()


def test_gloo_peer_group_setup_failure_raises_on_every_rank():
    """A rank whose mailbox set-up fails still joins the handle exchange, so no
    rank blocks, and every rank raises (bench.py then falls back to NCCL)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"{os.getpid()}f{port}"
    ps = [ctx.Process(target=_worker_peer_fail, args=(r, world, port, tag, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert set(res.values()) == {"raised"}, res
