"""GPU parity of the segmented kernel's guided multi-segment batches (the
production path of BASELINE config 5) and of the batched entry point at the
sizes where a warp reduces up to 255 rows per batch; and all 2^20 outputs of
the full-size C5 workload, element by element against the exact oracle.

The union-stream kernel (csrc/tcr_segmented.cu) hands out batches of several
consecutive segments only while S > hint + 2 * total_warps * batch (~75 776
CSR segments, ~2.4 M rows of L <= 128 on a 148-SM B200); below that every
batch holds one segment.  These tests are sized past that switch, so the
intra-batch segment transitions (segment ends inside a tile, runs of empty
segments, trailing empty segments of a batch) run many times.  Each segment
is the paper's group decomposition with a zero-padded trailing group
(§IV.A) applied to [off[j], off[j+1]).
"""
import os

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

pytestmark = pytest.mark.gpu
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))
DTYPES = ["f16", "bf16", "e4m3", "e5m2"]


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    return m


def _gen_device(dtype, seed, n, dist, xoff):
    """Bits of the (seed, dist) stream for ``dtype`` at a misaligned device
    address (``xoff`` elements past a 256-byte aligned allocation), and the
    same bits on the host (the device generator equals the host definition:
    test_gpu_segmented.py / test_gpu_fp8.py)."""
    import torch

    if dtype in ("e4m3", "e5m2"):
        fmt = gen.FP8_E4M3 if dtype == "e4m3" else gen.FP8_E5M2
        src = gen.generate_tensor_fp8(seed, 0, n, dist, fmt).view(torch.uint8)
        buf = torch.empty(n + xoff + 16, dtype=torch.uint8, device="cuda")
        tdt = torch.float8_e4m3fn if dtype == "e4m3" else torch.float8_e5m2
    else:
        src = gen.generate_tensor(seed, 0, n, dist, bf16=dtype == "bf16").view(torch.int16)
        buf = torch.empty(n + xoff + 8, dtype=torch.int16, device="cuda")
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    x = buf[xoff:xoff + n]
    x.copy_(src)
    del src
    host = x.cpu().numpy()
    host = host.view(np.uint8) if dtype in ("e4m3", "e5m2") else host.view(np.uint16)
    return x.view(tdt), host


def _oracle_ok(dtype, bits, off, g):
    """ok[j] = within_tolerance(g[j], exact R of segment j), every segment."""
    if dtype == "f16":
        return oracle.within_tolerance_segments(
            g, oracle.exact_segment_sums_fp16_array(bits, off, threads=THREADS))
    if dtype in ("e4m3", "e5m2"):
        fmt = oracle.FP8_E4M3 if dtype == "e4m3" else oracle.FP8_E5M2
        return oracle.within_tolerance_segments(
            g, oracle.exact_segment_sums_fp8_array(bits, off, fmt, threads=THREADS))
    es = oracle.exact_segment_sums_bf16(bits, off)
    return np.array([oracle.within_tolerance(float(g[j]), es[j]) for j in range(len(es))])


def _run_csr(tcr, x, off_t, S, algo):
    import torch

    out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
    tcr.tcr_reduce_sum_segmented_ex(x, off_t, out, algo=algo)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
@pytest.mark.parametrize("dtype", DTYPES)
def test_csr_guided_batches_vs_oracle(tcr, dtype, algo):
    """S = 2^17 + 77 CSR segments, lengths 0..20000 (a quarter empty, a
    quarter 1..7, tile-crossing, long), misaligned x and offsets: every
    output vs the oracle, empty segments exactly +0.0, integer data
    bitwise, and a second launch bitwise identical."""
    import torch

    S = (1 << 17) + 77
    lens = gen.mixed_lengths(1700 + len(dtype), S)
    start = 5
    off = gen.offsets_from_lengths(lens, start=start)
    n = int(off[-1]) + 11
    x, bits = _gen_device(dtype, 31, n, gen.UNIFORM_PM1, xoff=3)
    off_t = torch.from_numpy(off).cuda()
    out = _run_csr(tcr, x, off_t, S, algo)
    g = out.cpu().numpy()
    ok = _oracle_ok(dtype, bits, off, g)
    bad = np.nonzero(~ok)[0]
    assert bad.size == 0, (bad[:8].tolist(), g[bad[:8]].tolist(), lens[bad[:8]].tolist())
    empty = lens == 0
    assert np.all(g[empty] == 0.0) and not np.any(np.signbit(g[empty]))
    assert torch.equal(out, _run_csr(tcr, x, off_t, S, algo))


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
def test_csr_guided_batches_integer_bitwise(tcr, algo):
    """SMALLINT data (integers in -2..2): every segment sum is an integer of
    magnitude <= 40000, exact in every precision the kernels use, so out[j]
    must equal the exact sum bitwise (catches an output written to the
    wrong j, or a piece of a tile counted twice / dropped, inside a batch)."""
    import torch

    S = (1 << 17) + 5
    lens = gen.mixed_lengths(99, S)
    off = gen.offsets_from_lengths(lens, start=1)
    n = int(off[-1]) + 3
    x, bits = _gen_device("f16", 77, n, gen.SMALLINT, xoff=1)
    out = _run_csr(tcr, x, torch.from_numpy(off).cuda(), S, algo)
    g = out.cpu().numpy()
    ss = oracle.exact_segment_sums_fp16_array(bits, off, threads=THREADS)
    want = ss.rec["t_lo"].view(np.int64).astype(np.float64) * 2.0 ** -24
    assert np.array_equal(g.astype(np.float64), want)


# (L, S): S past the switch where batches reach 255 (L = 1, 7), 163 (L = 100)
# and 49 (L = 333) rows
BATCHED = [(1, 4_000_000), (7, 4_000_000), (100, 2_500_000), (333, 1_000_000)]


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
@pytest.mark.parametrize("L,S", BATCHED)
def test_batched_guided_vs_oracle(tcr, L, S, algo):
    import torch

    n = L * S
    for dtype, xoff in (("f16", 3), ("e4m3", 5)):
        if dtype == "e4m3" and L == 100:
            continue  # one fp8 case per row length suffices beyond L in {1, 7, 333}
        x, bits = _gen_device(dtype, 500 + L, n + 9, gen.UNIFORM_PM1, xoff=xoff)
        out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
        tcr.tcr_reduce_sum_batched_ex(x, L, out, algo=algo)
        torch.cuda.synchronize()
        g = out.cpu().numpy()
        off = np.arange(S + 1, dtype=np.int64) * L
        ok = _oracle_ok(dtype, bits, off, g)
        bad = np.nonzero(~ok)[0]
        assert bad.size == 0, (dtype, bad[:8].tolist(), g[bad[:8]].tolist())
        out2 = torch.empty_like(out)
        tcr.tcr_reduce_sum_batched_ex(x, L, out2, algo=algo)
        torch.cuda.synchronize()
        assert torch.equal(out, out2)
        del x, out, out2


def test_full_size_c5_all_outputs(tcr):
    """BASELINE config 5 at full size (2^20 log-uniform segments, ~1.24e10
    elements, 24.7 GB), in the launch configuration bench.py times: all 2^20
    outputs of the MMA path and of the shuffle path vs the exact oracle,
    element by element (x copied back in chunks of 2^16 segments)."""
    import torch

    S = 1 << 20
    lens = gen.loguniform_lengths(gen.SEED_C5, S)
    off = gen.offsets_from_lengths(lens)
    n = int(off[-1])
    x = gen.generate_tensor(gen.SEED_C5, 0, n, gen.UNIFORM_PM1)
    toff = torch.from_numpy(off).cuda()
    outs = {}
    for algo, f in (("mma", tcr.tcr_reduce_sum_segmented),
                    ("shuffle", tcr.tcr_reduce_sum_segmented_shuffle)):
        out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
        f(x, toff, out)
        torch.cuda.synchronize()
        outs[algo] = out.cpu().numpy()
    chunk = 1 << 16
    for j0 in range(0, S, chunk):
        j1 = min(S, j0 + chunk)
        a, b = int(off[j0]), int(off[j1])
        bits = x[a:b].view(torch.int16).cpu().numpy().view(np.uint16)
        ss = oracle.exact_segment_sums_fp16_array(bits, off[j0:j1 + 1] - a, threads=THREADS)
        for algo, g in outs.items():
            ok = oracle.within_tolerance_segments(g[j0:j1], ss)
            bad = np.nonzero(~ok)[0]
            assert bad.size == 0, (algo, (bad[:8] + j0).tolist())
        del bits
    del x


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_batched_rows_as_mma_rows(tcr, dtype):
    """Fixed-length rows with L % 32 == 0, L <= 2048 and a 16-byte aligned x
    take the rows-as-MMA-rows kernel (16 segments fill the 16 rows of A, the
    row sums of Eq. 10 are the segment sums): every row vs the oracle, ragged
    last slab (S % 16 != 0), integer data bitwise, and the same rows through
    a misaligned x (the union-stream kernel) agree within tolerance."""
    import torch

    for L, S in ((32, 100_003), (64, 40_001), (96, 33_333), (224, 20_000), (256, 65_541),
                 (480, 9_999), (2048, 1_029)):
        n = L * S
        x, bits = _gen_device(dtype, 900 + L, n, gen.UNIFORM_PM1, xoff=0)
        assert x.data_ptr() % 16 == 0
        out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
        tcr.tcr_reduce_sum_batched_ex(x, L, out, algo="mma_sync")
        torch.cuda.synchronize()
        g = out.cpu().numpy()
        ok = _oracle_ok(dtype, bits, np.arange(S + 1, dtype=np.int64) * L, g)
        assert ok.all(), (L, np.nonzero(~ok)[0][:8].tolist())
        if dtype == "f16":
            xi, bi = _gen_device(dtype, 77, n, gen.SMALLINT, xoff=0)
            tcr.tcr_reduce_sum_batched_ex(xi, L, out, algo="mma_sync")
            torch.cuda.synchronize()
            ss = oracle.exact_segment_sums_fp16_array(bi, np.arange(S + 1, dtype=np.int64) * L,
                                                      threads=THREADS)
            want = ss.rec["t_lo"].view(np.int64).astype(np.float64) * 2.0 ** -24
            assert np.array_equal(out.cpu().numpy().astype(np.float64), want), L
