"""GPU tests of NEXT-2, the cross-GPU combine fused into the reduction kernel
(tcr_reduce_sum_peer, csrc/tcr_peer.cuh).

This box has ONE GPU, and kernels of separate launches must never wait on
one another on one GPU (B200_PROFILING.md).  The multi-rank protocol is
therefore exercised as the guide prescribes: all ranks emulated in ONE
cooperative launch (tcr_reduce_sum_peer_emulated: grid slice r = rank r, the
same kernel and the same push / wait / rank-ordered sum), plus the real
single-process entry at nranks = 1, the timeout path (a peer that never
comes), and CUDA IPC mappings of a second process's mailbox used inside the
emulated launch.  The host logic of PeerGroup is covered under gloo in
tests/test_multigpu_gloo.py.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import tcr_inputs as gen
from exact_state_decode import exact_limbs_to_int

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    return m


@pytest.fixture
def mailboxes(tcr):
    boxes = [tcr.tcr_peer_mailbox_alloc() for _ in range(tcr.TCR_MAX_PEERS)]
    yield boxes
    import torch

    torch.cuda.synchronize()
    for b in boxes:
        tcr.tcr_peer_mailbox_free(b)


def _dev(bits):
    import torch

    return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.float16)


def _shards(n, P):
    return [(n * r // P, n * (r + 1) // P) for r in range(P)]


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle", "tcgen05"])
@pytest.mark.parametrize("n", [0, 1, 4097, 1_000_003, (1 << 29) + 7])
def test_single_rank_equals_f64_entry(tcr, mailboxes, algo, n):
    """nranks = 1: the fused kernel is the ordinary reduction plus 0.0 + v
    (compared at the peer variant's fixed unroll of 4, so both launches use
    the same grid and chain)."""
    import torch

    x = (_dev(gen.generate(3, 0, n, gen.UNIFORM_PM1)) if n <= (1 << 24)
         else gen.generate_tensor(3, 0, n, gen.UNIFORM_PM1))  # 1 GiB: the tcgen05 1-CTA/SM shape
    ref = torch.empty(1, dtype=torch.float64, device="cuda")
    tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 4)
    try:
        tcr.tcr_reduce_sum_ex(x, out_f64=ref, algo=algo)
    finally:
        tcr.tcr_set_config(tcr.TCR_CFG_UNROLL, 0)
    o64 = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    for _ in range(3):  # consecutive epochs on the same mailbox
        tcr.tcr_reduce_sum_peer(x, mailboxes[:1], 0, out_f32=o32, out_f64=o64, algo=algo)
        torch.cuda.synchronize()
        assert o64.item() == ref.item()
        assert o32.item() == float(np.float32(ref.item()))
    assert not tcr.tcr_peer_mailbox_error(mailboxes[0])


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", ["mma_sync", "shuffle", "tcgen05"])
def test_emulated_ranks(tcr, mailboxes, P, algo):
    import torch

    n = 3_000_017
    o32 = torch.full((P,), float("nan"), dtype=torch.float32, device="cuda")
    o64 = torch.full((P,), float("nan"), dtype=torch.float64, device="cuda")
    for epoch, dist in enumerate((gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01, gen.SMALLINT)):
        bits = gen.generate(40 + epoch, 0, n, dist)
        tcr.tcr_reduce_sum_peer_emulated(_dev(bits), mailboxes[:P], out_f32=o32, out_f64=o64,
                                         algo=algo)
        torch.cuda.synchronize()
        g32, g64 = o32.cpu().tolist(), o64.cpu().tolist()
        assert len(set(g64)) == 1 and len(set(g32)) == 1, (epoch, g64)  # replicated, bitwise
        es = oracle.exact_sum_fp16(bits)
        assert oracle.within_tolerance(g32[0], es), (epoch, g32[0], es.f64())
        if dist == gen.SMALLINT:  # integer data: every partial and the total are exact
            assert g64[0] == es.f64() and g32[0] == es.f32()
    for b in mailboxes[:P]:
        assert not tcr.tcr_peer_mailbox_error(b)


def test_emulated_partials_are_the_ranks_shard_sums(tcr, mailboxes):
    """One-hot data: the total is exactly the sum of per-shard contributions,
    and a shard boundary off by one element would double count or drop."""
    import torch

    P, n = 8, 1 << 20
    o64 = torch.empty(P, dtype=torch.float64, device="cuda")
    for lo, hi in _shards(n, P):
        for pos in (lo, hi - 1):
            bits = np.zeros(n, dtype=np.uint16)
            bits[pos] = 0x3C00
            tcr.tcr_reduce_sum_peer_emulated(_dev(bits), mailboxes[:P], out_f64=o64)
            torch.cuda.synchronize()
            assert o64.cpu().tolist() == [1.0] * P, pos


@pytest.mark.parametrize("algo", ["default", "tcgen05"])
def test_emulated_bf16_fp8(tcr, mailboxes, algo):
    import torch

    P, n = 4, 500_003
    out = torch.empty(P, dtype=torch.float32, device="cuda")
    b = gen.generate_bf16(5, 0, n, gen.UNIFORM_PM1)
    xb = torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
    tcr.tcr_reduce_sum_peer_emulated(xb, mailboxes[:P], out_f32=out, algo=algo)
    torch.cuda.synchronize()
    assert len(set(out.cpu().tolist())) == 1
    assert oracle.within_tolerance(out[0].item(), oracle.exact_sum_bf16(b))
    f8 = gen.generate_fp8(5, 0, n, gen.UNIFORM_PM1, gen.FP8_E4M3)
    x8 = torch.from_numpy(f8).cuda().view(torch.float8_e4m3fn)
    tcr.tcr_reduce_sum_peer_emulated(x8, mailboxes[:P], out_f32=out, algo=algo)
    torch.cuda.synchronize()
    assert len(set(out.cpu().tolist())) == 1
    assert oracle.within_tolerance(out[0].item(), oracle.exact_sum_fp8(f8, gen.FP8_E4M3))


def test_emulated_c4_scale(tcr, mailboxes):
    """BASELINE config 4 at its full size (2^33 elements, 16 GiB, 8 ranks)
    emulated in one launch: all-ones data makes the exact answer n, and the
    fp64 combine of the 8 exact partials is exact."""
    import torch

    n, P = 1 << 33, 8
    x = gen.generate_tensor(gen.SEED_C4, 0, n, gen.ONES)
    o64 = torch.empty(P, dtype=torch.float64, device="cuda")
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    # both fused kernels: tcgen05 (r02) and mma.sync
    for algo in ("tcgen05", "mma_sync"):
        o64.fill_(float("nan"))
        o32.fill_(float("nan"))
        tcr.tcr_reduce_sum_peer_emulated(x, mailboxes[:P], out_f32=o32, out_f64=o64, algo=algo)
        torch.cuda.synchronize()
        assert o64.cpu().tolist() == [float(n)] * P, algo
        assert o32.cpu().tolist() == [float(n)] * P, algo
    del x


def test_graph_replay_advances_the_device_epoch(tcr, mailboxes):
    """The epoch lives in the mailbox, so a captured launch replays correctly
    with fresh data (a host-side epoch baked into the graph would read the
    previous replay's partials)."""
    import torch

    P, n = 4, 200_003
    x = torch.empty(n, dtype=torch.float16, device="cuda")
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    x.copy_(_dev(gen.generate(1, 0, n, gen.SMALLINT)))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):  # warm-up: the stream's workspace exists before capture
        tcr.tcr_reduce_sum_peer_emulated(x, mailboxes[:P], out_f64=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        tcr.tcr_reduce_sum_peer_emulated(x, mailboxes[:P], out_f64=out,
                                         stream=torch.cuda.current_stream())
    for seed in range(2, 7):
        bits = gen.generate(seed, 0, n, gen.SMALLINT)
        x.copy_(_dev(bits))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert out.cpu().tolist() == [oracle.exact_sum_fp16(bits).f64()] * P, seed


def test_timeout_when_a_peer_never_arrives(tcr, mailboxes):
    """Rank 0 of a 2-rank group whose rank 1 never calls: the wait is bounded
    (here 100 ms), the result is NaN and the error word is set; reset clears
    it.  (A single launch waiting for nothing -- no second kernel involved.)"""
    import math

    import torch

    old = tcr.tcr_get_config(tcr.TCR_CFG_PEER_TIMEOUT_MS)
    tcr.tcr_set_config(tcr.TCR_CFG_PEER_TIMEOUT_MS, 100)
    try:
        x = _dev(gen.generate(1, 0, 10_000, gen.UNIFORM_PM1))
        out = torch.zeros(1, dtype=torch.float32, device="cuda")
        tcr.tcr_reduce_sum_peer(x, mailboxes[:2], 0, out_f32=out)
        torch.cuda.synchronize()
        assert math.isnan(out.item())
        assert tcr.tcr_peer_mailbox_error(mailboxes[0])
        for b in mailboxes[:2]:
            tcr.tcr_peer_mailbox_reset(b)
        torch.cuda.synchronize()
        assert not tcr.tcr_peer_mailbox_error(mailboxes[0])
        tcr.tcr_reduce_sum_peer_emulated(x, mailboxes[:2], out_f32=torch.empty(2, device="cuda"))
        torch.cuda.synchronize()
        assert not tcr.tcr_peer_mailbox_error(mailboxes[0])
    finally:
        tcr.tcr_set_config(tcr.TCR_CFG_PEER_TIMEOUT_MS, old)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, port, q):
    import torch
    import torch.distributed as dist

    import bench

    bench.wait_for_cuda_driver()
    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as tcr

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    own = tcr.tcr_peer_mailbox_alloc()
    handles = [None, None]
    dist.all_gather_object(handles, tcr.tcr_peer_ipc_handle(own))
    if rank == 0:
        # ONE emulated 2-rank launch in this process: rank 1's mailbox is the
        # other process's allocation, mapped through CUDA IPC.  Nothing in
        # process 1 waits on the GPU.
        peer = tcr.tcr_peer_ipc_open(handles[1])
        bits = gen.generate(9, 0, 777_777, gen.SMALLINT)
        x = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.float16)
        out = torch.empty(2, dtype=torch.float64, device="cuda")
        tcr.tcr_reduce_sum_peer_emulated(x, [own, peer], out_f64=out)
        torch.cuda.synchronize()
        q.put(("result", out.cpu().tolist(), oracle.exact_sum_fp16(bits).f64()))
        tcr.tcr_peer_ipc_close(peer)
    dist.barrier()
    if rank == 1:
        q.put(("peer_error", tcr.tcr_peer_mailbox_error(own)))
    dist.barrier()
    tcr.tcr_peer_mailbox_free(own)
    dist.destroy_process_group()


def test_ipc_mapped_mailbox_in_fused_kernel(tcr):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    msgs = dict((m[0], m[1:]) for m in (q.get(timeout=240) for _ in range(2)))
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    vals, want = msgs["result"]
    assert vals == [want, want]
    assert msgs["peer_error"] == (False,)


# ---------------- NEXT-2 x NEXT-3: the exact limb combine ----------------

@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_exact_emulated_bitwise(tcr, mailboxes, P):
    """The fused exact combine: every rank's result is the correctly rounded
    exact sum, bit for bit, and the summed limbs are the oracle's integer."""
    import torch

    acc = torch.empty(6 * P, dtype=torch.int64, device="cuda")
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    o64 = torch.empty(P, dtype=torch.float64, device="cuda")
    for seed, n, dist in ((1, 3_000_017, gen.WIDE), (2, 777, gen.UNIFORM_PM1),
                          (3, 1 << 22, gen.UNIFORM_01), (4, 5, gen.SMALLINT)):
        bits = gen.generate(seed, 0, n, dist)
        es = oracle.exact_sum_fp16(bits)
        tcr.tcr_reduce_sum_exact_peer_emulated(_dev(bits), mailboxes[:P], acc=acc, out_f32=o32,
                                               out_f64=o64)
        torch.cuda.synchronize()
        assert o32.cpu().tolist() == [es.f32()] * P, (seed, P)
        assert o64.cpu().tolist() == [es.f64()] * P, (seed, P)
        for r in range(P):
            assert exact_limbs_to_int(acc[6 * r:6 * r + 6]) == es.T


def test_exact_single_rank_equals_exact_entry(tcr, mailboxes):
    import torch

    bits = gen.generate(8, 0, 1_234_567, gen.WIDE)
    x = _dev(bits)
    a = torch.empty(6, dtype=torch.int64, device="cuda")
    b = torch.empty(6, dtype=torch.int64, device="cuda")
    tcr.tcr_reduce_sum_exact(x, acc=a)
    tcr.tcr_reduce_sum_exact_peer(x, mailboxes[:1], 0, acc=b)
    torch.cuda.synchronize()
    assert exact_limbs_to_int(a) == exact_limbs_to_int(b)


def test_exact_and_fp64_combines_interleave(tcr, mailboxes):
    """Both kinds of combine advance the same device epoch: alternating them
    on one group stays consistent."""
    import torch

    P = 4
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    for i in range(6):
        bits = gen.generate(50 + i, 0, 100_003, gen.SMALLINT)
        es = oracle.exact_sum_fp16(bits)
        if i % 2:
            tcr.tcr_reduce_sum_exact_peer_emulated(_dev(bits), mailboxes[:P], out_f32=o32)
        else:
            tcr.tcr_reduce_sum_peer_emulated(_dev(bits), mailboxes[:P], out_f32=o32)
        torch.cuda.synchronize()
        assert o32.cpu().tolist() == [es.f32()] * P, i
    assert not any(tcr.tcr_peer_mailbox_error(b) for b in mailboxes[:P])


def test_exact_specials_in_one_shard(tcr, mailboxes):
    import math

    import torch

    P, n = 4, 10_000
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    for special, expect in ((0x7C00, math.inf), (0xFC00, -math.inf), (0x7E00, math.nan)):
        bits = gen.generate(9, 0, n, gen.UNIFORM_PM1)
        bits[n - 3] = special  # lands in the last rank's shard
        tcr.tcr_reduce_sum_exact_peer_emulated(_dev(bits), mailboxes[:P], out_f32=o32)
        torch.cuda.synchronize()
        for g in o32.cpu().tolist():
            assert (math.isnan(g) if math.isnan(expect) else g == expect), (special, g)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_exact_bulk_peer_emulated_bitwise(tcr, mailboxes, P):
    """The TMA-fed exact kernel fused with the limb combine (TCR_CFG_EXACT_BULK
    = 2 forces it below its 128 MiB-per-rank threshold; r02 §18): bitwise
    equal to the oracle on every rank, static and dynamic tails, and equal to
    the LDG peer kernel's limbs."""
    import torch

    keys = (tcr.TCR_CFG_EXACT_BULK, tcr.TCR_CFG_TC05_DYN_MIN_RUN)
    saved = [tcr.tcr_get_config(k) for k in keys]
    acc = torch.empty(6 * P, dtype=torch.int64, device="cuda")
    o32 = torch.empty(P, dtype=torch.float32, device="cuda")
    o64 = torch.empty(P, dtype=torch.float64, device="cuda")
    try:
        for seed, n, dist in ((1, 3_000_017, gen.WIDE), (3, (1 << 24) + 9, gen.UNIFORM_01), (4, 5, gen.SMALLINT)):
            bits = gen.generate(seed, 0, n, dist)
            es = oracle.exact_sum_fp16(bits)
            for eb, mr in ((2, 32), (2, 0), (0, 32)):
                tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
                tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, mr)
                tcr.tcr_reduce_sum_exact_peer_emulated(_dev(bits), mailboxes[:P], acc=acc, out_f32=o32,
                                                       out_f64=o64)
                torch.cuda.synchronize()
                assert o32.cpu().tolist() == [es.f32()] * P, (seed, P, eb, mr)
                assert o64.cpu().tolist() == [es.f64()] * P, (seed, P, eb, mr)
                for r in range(P):
                    assert exact_limbs_to_int(acc[6 * r:6 * r + 6]) == es.T, (seed, P, eb, mr, r)
        for b in mailboxes[:P]:
            assert not tcr.tcr_peer_mailbox_error(b)
    finally:
        for k, v in zip(keys, saved):
            tcr.tcr_set_config(k, v)
