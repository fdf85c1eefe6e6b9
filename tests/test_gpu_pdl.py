"""Programmatic dependent launch (TCR_CFG_PDL, r02) under stress: long runs
of back-to-back launches on one stream, where a call's CTAs are scheduled
while the previous kernel drains.  Every result must equal, bit for bit, the
result of the same call made alone (the kernels are deterministic), and be
within tolerance of the exact oracle.  This catches a call that reads its
input, the completion ticket or the segment scheduler's counters before the
previous kernel on the stream has finished with them."""
import numpy as np
import pytest

import oracle
import tcr_inputs as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    assert m.tcr_get_config(m.TCR_CFG_PDL) == 1  # the default under test
    return m


def _x(seed, n, dist=gen.UNIFORM_PM1):
    return gen.generate_tensor(seed, 0, n, dist), gen.generate(seed, 0, n, dist)


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle", "default"])
def test_flat_back_to_back_alternating_sizes(tcr, algo):
    """300 launches alternating a one-CTA size, a one-wave size and a
    multi-wave size (different grids, same workspace and ticket)."""
    import torch

    cases = [_x(11, (1 << 16) + 37), _x(12, (1 << 22) + 5), _x(13, (1 << 26) + 3)]
    alone = []
    for x, _ in cases:
        o = torch.empty(1, dtype=torch.float32, device="cuda")
        tcr.tcr_reduce_sum_ex(x, out_f32=o, algo=algo)
        torch.cuda.synchronize()
        alone.append(float(o.item()))
    for (x, bits), g in zip(cases, alone):
        assert oracle.within_tolerance(g, oracle.exact_sum_fp16(bits, threads=8))
    K = 300
    outs = torch.full((K,), float("nan"), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(K):
            tcr.tcr_reduce_sum_ex(cases[i % 3][0], out_f32=outs[i:i + 1], algo=algo, stream=s)
    torch.cuda.synchronize()
    got = outs.cpu().numpy()
    for i in range(K):
        assert got[i] == np.float32(alone[i % 3]), (i, got[i], alone[i % 3])


def test_input_written_by_the_previous_kernel(tcr):
    """x is rewritten by a torch copy right before every reduction (a
    primary without PDL): each result must be the sum of the data just
    written, never of the previous contents."""
    import torch

    n = (1 << 22) + 9
    srcs = [gen.generate_tensor(20 + k, 0, n, gen.SMALLINT) for k in range(4)]
    want = [oracle.exact_sum_fp16(gen.generate(20 + k, 0, n, gen.SMALLINT), threads=8).f32()
            for k in range(4)]
    assert len(set(want)) == 4
    x = torch.empty(n, dtype=torch.float16, device="cuda")
    K = 200
    outs = torch.empty(K, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(K):
            x.copy_(srcs[i % 4])
            tcr.tcr_reduce_sum_ex(x, out_f32=outs[i:i + 1], algo="mma_sync", stream=s)
    torch.cuda.synchronize()
    got = outs.cpu().numpy()
    for i in range(K):
        assert got[i] == np.float32(want[i % 4]), (i, got[i], want[i % 4])


def test_segmented_and_batched_back_to_back(tcr):
    """CSR (scheduler counters reset by the last warp of the previous
    launch), fixed-length rows as MMA rows and the whole-tile rows kernel,
    interleaved with flat reductions on one stream, 60 rounds."""
    import torch

    S = 50_000
    lens = gen.mixed_lengths(5, S)
    off = gen.offsets_from_lengths(lens)
    n = int(off[-1])
    xs, bits_s = _x(31, n)
    toff = torch.from_numpy(off).cuda()
    xb64, bits64 = _x(32, 64 * 40_000)
    xb1k, bits1k = _x(33, 1024 * 3_000)
    xf, bits_f = _x(34, (1 << 20) + 1)

    def run(stream, o_seg, o_b64, o_b1k, o_f):
        tcr.tcr_reduce_sum_segmented_ex(xs, toff, o_seg, stream=stream)
        tcr.tcr_reduce_sum_batched_ex(xb64, 64, o_b64, stream=stream)
        tcr.tcr_reduce_sum_ex(xf, out_f32=o_f, stream=stream)
        tcr.tcr_reduce_sum_batched_ex(xb1k, 1024, o_b1k, stream=stream)

    mk = lambda m: torch.full((m,), float("nan"), dtype=torch.float32, device="cuda")  # noqa: E731
    ref = [mk(S), mk(40_000), mk(3_000), mk(1)]
    run(torch.cuda.current_stream(), *ref)
    torch.cuda.synchronize()
    ok = oracle.within_tolerance_segments(ref[0].cpu().numpy(), oracle.exact_segment_sums_fp16_array(
        bits_s, off, threads=8))
    assert ok.all()
    ok = oracle.within_tolerance_segments(ref[1].cpu().numpy(), oracle.exact_segment_sums_fp16_array(
        bits64, np.arange(40_001, dtype=np.int64) * 64, threads=8))
    assert ok.all()
    ok = oracle.within_tolerance_segments(ref[2].cpu().numpy(), oracle.exact_segment_sums_fp16_array(
        bits1k, np.arange(3_001, dtype=np.int64) * 1024, threads=8))
    assert ok.all()
    assert oracle.within_tolerance(float(ref[3].item()), oracle.exact_sum_fp16(bits_f))
    R = 60
    outs = [[mk(S), mk(40_000), mk(3_000), mk(1)] for _ in range(R)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(R):
            run(s, *outs[r])
    torch.cuda.synchronize()
    for r in range(R):
        for a, b in zip(outs[r], ref):
            assert torch.equal(a, b), r


def test_pdl_off_gives_identical_results(tcr):
    """TCR_CFG_PDL = 0 (plain launches) and 1 give bitwise identical outputs."""
    import torch

    x, _ = _x(41, (1 << 24) + 77)
    res = {}
    for pdl in (0, 1):
        tcr.tcr_set_config(tcr.TCR_CFG_PDL, pdl)
        try:
            o = torch.empty(8, dtype=torch.float32, device="cuda")
            for i in range(8):
                tcr.tcr_reduce_sum_ex(x, out_f32=o[i:i + 1])
            torch.cuda.synchronize()
            res[pdl] = o.cpu().numpy()
        finally:
            tcr.tcr_set_config(tcr.TCR_CFG_PDL, 1)
    assert np.array_equal(res[0], res[1]) and len(set(res[1].tolist())) == 1
