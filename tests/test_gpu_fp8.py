"""NEXT-4: fp8 (E4M3 / E5M2) inputs through the MMA encoding (mma.sync: the
exact binary16 conversion of each tile as two m16n8k16 against ones; tcgen05
kind::f8f6f4, B = fp8 ones) and the shuffle path, vs the
exact fp8 oracle; tolerance |g - R| <= 2^-20 * sum|x_i|; any byte alignment."""
import numpy as np
import pytest

import oracle
import tcr_inputs as gen
from exact_state_decode import exact_limbs_to_int, exact_bf16_windows_to_value

pytestmark = pytest.mark.gpu
ALGOS = ["mma_sync", "tcgen05", "shuffle", "bulk"]
FMTS = [oracle.FP8_E4M3, oracle.FP8_E5M2]


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    return m


def _dev(bits, offset, fmt):
    import torch

    buf = torch.empty(bits.size + offset + 16, dtype=torch.uint8, device="cuda")
    x = buf[offset:offset + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits))
    return x.view(torch.float8_e4m3fn if fmt == oracle.FP8_E4M3 else torch.float8_e5m2)


def _sum(tcr, x, algo):
    import torch

    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    tcr.tcr_reduce_sum_ex(x, out_f32=o32, algo=algo)
    torch.cuda.synchronize()
    return float(o32.item())


@pytest.mark.parametrize("fmt", FMTS)
def test_device_generator_matches_host(tcr, fmt):
    import torch

    for dist in range(6):
        d = gen.generate_tensor_fp8(41 + dist, 777, 100_003, dist, fmt)
        assert np.array_equal(d.view(torch.uint8).cpu().numpy(),
                              gen.generate_fp8(41 + dist, 777, 100_003, dist, fmt)), dist


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("dist", [gen.UNIFORM_PM1, gen.UNIFORM_01, gen.WIDE, gen.ALTERNATING, gen.ONES])
def test_fp8_sizes_dists_alignment(tcr, algo, fmt, dist):
    for n in (0, 1, 15, 16, 17, 511, 512, 513, 40_000, (1 << 22) + 7):
        bits = gen.generate_fp8(300 + dist, 0, n, dist, fmt)
        es = oracle.exact_sum_fp8(bits, fmt)
        for off in (0, 1, 9):
            g = _sum(tcr, _dev(bits, off, fmt), algo)
            assert oracle.within_tolerance(g, es), (algo, fmt, dist, n, off, g, es.f64())
        if dist == gen.ONES:
            assert g == float(n)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("fmt", FMTS)
def test_fp8_integers_bitwise_and_deterministic(tcr, algo, fmt):
    bits = gen.generate_fp8(5, 0, (1 << 22) + 3, gen.SMALLINT, fmt)
    es = oracle.exact_sum_fp8(bits, fmt)
    x = _dev(bits, 3, fmt)
    g = _sum(tcr, x, algo)
    assert g == float(es.value)
    assert g == _sum(tcr, x, algo)


@pytest.mark.parametrize("fmt", FMTS)
def test_fp8_full_size(tcr, fmt):
    import torch

    n = 1 << 31  # 2 GiB of fp8
    x = gen.generate_tensor_fp8(gen.SEED_C3, 0, n, gen.UNIFORM_PM1, fmt)
    bits = x.view(torch.uint8)
    es = oracle.ExactSum(0, 0, unit_exp={0: -9, 1: -16}[fmt])
    for lo in range(0, n, 1 << 28):
        es = es + oracle.exact_sum_fp8(bits[lo:lo + (1 << 28)].cpu().numpy(), fmt)
    for algo in ALGOS:
        g = _sum(tcr, x, algo)
        assert oracle.within_tolerance(g, es), (algo, g, es.f64())


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
def test_fp8_segmented_edges_and_mix(tcr, fmt, algo):
    """CSR segments of fp8: every segment vs the exact fp8 oracle, with
    lengths around the 16-element vector and 512-element tile boundaries,
    empty segments, odd byte offsets, and a log-uniform mix."""
    import torch

    lens = [0, 1, 2, 15, 16, 17, 31, 511, 512, 513, 0, 1023, 1024, 1025, 8191, 65536, 3, 0, 70001]
    lens = np.array(lens + list(gen.loguniform_lengths(5, 500)), dtype=np.int64)
    for start in (0, 5, 17):
        off = gen.offsets_from_lengths(lens, start=start)
        bits = gen.generate_fp8(31 + start, 0, int(off[-1]) + 7, gen.WIDE, fmt)
        for xoff in (0, 3):
            out = torch.full((len(lens),), float("nan"), dtype=torch.float32, device="cuda")
            tcr.tcr_reduce_sum_segmented_ex(_dev(bits, xoff, fmt), torch.from_numpy(off).cuda(), out,
                                            algo=algo)
            torch.cuda.synchronize()
            g = out.cpu().numpy()
            for j in range(len(lens)):
                es = oracle.exact_sum_fp8(bits[off[j]:off[j + 1]], fmt)
                assert oracle.within_tolerance(float(g[j]), es), (start, xoff, j, g[j], es.f64())
                if lens[j] == 0:
                    assert g[j] == 0.0


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
def test_fp8_batched(tcr, fmt, algo):
    """Fixed-length fp8 rows: L = 512 * T takes the whole-tile rows kernel
    (16-byte-aligned x), other L and misaligned x the union-stream kernel."""
    import torch

    for L, S in ((512, 3000), (1024, 999), (2048, 300), (4096, 129), (511, 777), (100, 5000),
                 (65536, 9)):
        bits = gen.generate_fp8(L, 0, L * S, gen.UNIFORM_PM1, fmt)
        ref = [oracle.exact_sum_fp8(bits[j * L:(j + 1) * L], fmt) for j in range(S)]
        for xoff in (0, 1):
            out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
            tcr.tcr_reduce_sum_batched_ex(_dev(bits, xoff, fmt), L, out, algo=algo)
            torch.cuda.synchronize()
            g = out.cpu().numpy()
            assert all(oracle.within_tolerance(float(g[j]), ref[j]) for j in range(S)), (L, S, xoff)


def test_fp8_segment_index_bit_exact(tcr):
    """All-ones fp8 data and pairwise-distinct lengths: out[j] == len(j) exactly."""
    import torch

    for fmt, one in ((oracle.FP8_E4M3, 0x38), (oracle.FP8_E5M2, 0x3C)):
        lens = np.random.default_rng(1).permutation(np.arange(0, 4000, 3))
        off = gen.offsets_from_lengths(lens, start=7)
        bits = np.full(int(off[-1]) + 16, one, dtype=np.uint8)
        out = torch.empty(len(lens), dtype=torch.float32, device="cuda")
        tcr.tcr_reduce_sum_segmented_ex(_dev(bits, 1, fmt), torch.from_numpy(off).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), lens.astype(np.float32))


@pytest.mark.parametrize("fmt", FMTS)
def test_fp8_exact_bitwise(tcr, fmt):
    """NEXT-3 x NEXT-4: tcr_reduce_sum_exact_ex on fp8 is bitwise equal to the
    exact fp8 oracle (every fp8 value is a binary16 value; same exact
    accumulation), for ragged sizes, every byte misalignment and all
    distributions; the limbs are the oracle's integer in units of 2^-24."""
    import torch

    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    acc = torch.empty(6, dtype=torch.int64, device="cuda")
    for n in (0, 1, 15, 16, 17, 511, 512, 513, 100_003, 3_000_017):
        for dist in (gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01, gen.SMALLINT):
            bits = gen.generate_fp8(n + dist, 0, n, dist, fmt)
            es = oracle.exact_sum_fp8(bits, fmt)
            for off in ((0, 1, 7) if n < 10_000 else (3,)):
                tcr.tcr_reduce_sum_exact_ex(_dev(bits, off, fmt), acc=acc, out_f32=o32, out_f64=o64)
                torch.cuda.synchronize()
                assert float(o32.item()) == es.f32(), (n, dist, off, o32.item(), es.f64())
                assert float(o64.item()) == es.f64(), (n, dist, off)
                T = exact_limbs_to_int(acc)
                assert T * oracle.UNIT == es.value, (n, dist, off)


def test_fp8_exact_specials(tcr):
    import math

    import torch

    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    cases = [(oracle.FP8_E4M3, 0x7F, "nan"), (oracle.FP8_E5M2, 0x7C, "+inf"),
             (oracle.FP8_E5M2, 0xFC, "-inf"), (oracle.FP8_E5M2, 0x7E, "nan")]
    for fmt, special, kind in cases:
        bits = gen.generate_fp8(1, 0, 5000, gen.UNIFORM_PM1, fmt)
        bits[1234] = special
        tcr.tcr_reduce_sum_exact_ex(_dev(bits, 0, fmt), out_f32=o32)
        torch.cuda.synchronize()
        g = float(o32.item())
        if kind == "nan":
            assert math.isnan(g), (fmt, special, g)
        else:
            assert g == (math.inf if kind == "+inf" else -math.inf), (fmt, special, g)


def test_exact_bf16_acc_state_is_mergeable(tcr):
    """The bfloat16 exact state (27 int64: 8 windows x 3 limbs + counts) holds
    the exact sum, and integer-summing the states of shards then finalizing
    gives the whole array's correctly rounded sum bitwise (as an int64 SUM
    allreduce across GPUs would)."""
    import torch

    n = 2_000_003
    bits = gen.generate_bf16(7, 0, n, gen.WIDE)
    es = oracle.exact_sum_bf16(bits)
    x = torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    W = tcr.TCR_EXACT_BF16_ACC_WORDS
    acc = torch.empty(W, dtype=torch.int64, device="cuda")
    tcr.tcr_reduce_sum_exact_ex(x, acc=acc)
    torch.cuda.synchronize()
    assert exact_bf16_windows_to_value(acc.cpu()) == es.value
    P = 3
    parts = torch.empty(P, W, dtype=torch.int64, device="cuda")
    for r in range(P):
        lo, hi = r * n // P, (r + 1) * n // P
        tcr.tcr_reduce_sum_exact_ex(x[lo:hi], acc=parts[r])
    tot = parts.sum(dim=0)  # the integer allreduce
    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    tcr.tcr_exact_finalize_ex(tot, tcr.TCR_DTYPE_BF16, out_f32=o32, out_f64=o64)
    torch.cuda.synchronize()
    assert float(o32.item()) == es.f32() and float(o64.item()) == es.f64()


def test_fp8_e4m3_exact_on_tcgen05(tcr):
    """The exact E4M3 entry from 64 MiB runs the tcgen05 dynamic-tail kernel
    (rows of 64 E4M3 values are exact in binary32, r02 §16) plus a NaN count:
    limbs, special counts and RNE outputs bitwise equal to the oracle, with
    and without NaNs (counted exactly), misaligned, static or dynamic tail,
    and equal to the LDG exact kernel's state (TCR_CFG_EXACT_BULK = 0)."""
    import torch

    fmt = oracle.FP8_E4M3
    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    acc = torch.empty(6, dtype=torch.int64, device="cuda")
    keys = (tcr.TCR_CFG_EXACT_BULK, tcr.TCR_CFG_TC05_DYN_MIN_RUN)
    saved = [tcr.tcr_get_config(k) for k in keys]
    try:
        for n in ((64 << 20) + 5, (1 << 29) + 32768 * 3 + 11):
            for dist in (gen.UNIFORM_PM1, gen.WIDE):
                bits = gen.generate_fp8(70 + dist, 0, n, dist, fmt)
                es = oracle.exact_sum_fp8(bits, fmt)
                for eb, mr in ((1, 32), (1, 0), (0, 32)):
                    tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, eb)
                    tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, mr)
                    acc.fill_(-7)
                    tcr.tcr_reduce_sum_exact_ex(_dev(bits, 3, fmt), acc=acc, out_f32=o32, out_f64=o64)
                    torch.cuda.synchronize()
                    a = acc.cpu().tolist()
                    assert exact_limbs_to_int(a) * oracle.UNIT == es.value, (n, dist, eb, mr)
                    assert a[3:] == [0, 0, 0] and 0 <= a[0] < (1 << 40) and 0 <= a[1] < (1 << 40)
                    assert float(o32.item()) == es.f32() and float(o64.item()) == es.f64(), (n, dist, eb)
        bits = gen.generate_fp8(7, 0, (64 << 20) + 3, gen.UNIFORM_PM1, fmt)
        bits[[5, len(bits) // 2, len(bits) - 2]] = [0x7F, 0xFF, 0x7F]  # three NaNs
        tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 1)
        for _ in range(2):  # the marker and the ticket reset between launches
            tcr.tcr_reduce_sum_exact_ex(_dev(bits, 0, fmt), acc=acc, out_f32=o32)
            torch.cuda.synchronize()
            a = acc.cpu().tolist()
            assert a[3:] == [3, 0, 0], a
            assert o32.item() != o32.item()
    finally:
        for k, v in zip(keys, saved):
            tcr.tcr_set_config(k, v)


@pytest.mark.parametrize("fmt", FMTS)
def test_fp8_exact_bulk_kernel_forced(tcr, fmt):
    """TCR_CFG_EXACT_BULK = 2 forces the TMA-fed exact kernel for fp8 too (below
    the 64 MiB E4M3 tcgen05 threshold): bitwise equal to the oracle, with the
    dynamic tail on at every size, misaligned, with a special value."""
    import torch

    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    acc = torch.empty(6, dtype=torch.int64, device="cuda")
    keys = (tcr.TCR_CFG_EXACT_BULK, tcr.TCR_CFG_TC05_DYN_MIN_RUN)
    saved = [tcr.tcr_get_config(k) for k in keys]
    try:
        tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 2)
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, 0)
        for n in (1, 32768 * 3 + 9, (1 << 24) + 77):
            bits = gen.generate_fp8(n, 0, n, gen.WIDE, fmt)
            es = oracle.exact_sum_fp8(bits, fmt)
            tcr.tcr_reduce_sum_exact_ex(_dev(bits, 5, fmt), acc=acc, out_f32=o32, out_f64=o64)
            torch.cuda.synchronize()
            assert exact_limbs_to_int(acc) * oracle.UNIT == es.value, (fmt, n)
            assert float(o32.item()) == es.f32() and float(o64.item()) == es.f64(), (fmt, n)
        bits = gen.generate_fp8(3, 0, 200_000, gen.UNIFORM_PM1, fmt)
        bits[100_000] = 0x7F  # NaN in both formats
        es = oracle.exact_sum_fp8(bits, fmt)
        tcr.tcr_reduce_sum_exact_ex(_dev(bits, 0, fmt), acc=acc, out_f32=o32)
        torch.cuda.synchronize()
        a = acc.cpu().tolist()
        assert (a[3], a[4], a[5]) == (es.n_nan, es.n_pinf, es.n_ninf), (fmt, a)
        assert o32.item() != o32.item()
    finally:
        for k, v in zip(keys, saved):
            tcr.tcr_set_config(k, v)
