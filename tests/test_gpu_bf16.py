"""NEXT-4: bfloat16 inputs through the same MMA encoding (mma.sync .bf16,
tcgen05 kind::f16 with BF16 operands) and the shuffle path, vs the exact
bfloat16 oracle; tolerance |g - R| <= 2^-20 * sum|x_i|."""
import numpy as np
import pytest

import oracle
import tcr_inputs as gen

pytestmark = pytest.mark.gpu
ALGOS = ["mma_sync", "tcgen05", "shuffle", "bulk"]


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    return m


def _dev(bits, offset=0):
    import torch

    buf = torch.empty(bits.size + offset + 8, dtype=torch.int16, device="cuda")
    x = buf[offset:offset + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits.view(np.int16)))
    return x.view(torch.bfloat16)


def _sum(tcr, x, algo):
    import torch

    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    o64 = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    tcr.tcr_reduce_sum_ex(x, out_f32=o32, out_f64=o64, algo=algo)
    torch.cuda.synchronize()
    return float(o32.item()), float(o64.item())


def test_device_generator_matches_host(tcr):
    import torch

    for dist in range(6):
        d = gen.generate_tensor(31 + dist, 12345, 100_003, dist, bf16=True)
        assert np.array_equal(d.view(torch.int16).cpu().numpy().view(np.uint16),
                              gen.generate_bf16(31 + dist, 12345, 100_003, dist)), dist


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dist", [gen.UNIFORM_PM1, gen.UNIFORM_01, gen.WIDE, gen.ALTERNATING, gen.ONES])
def test_bf16_sizes_and_dists(tcr, algo, dist):
    for n in (0, 1, 7, 257, 8193, 65536 + 37, (1 << 22) + 123):
        bits = gen.generate_bf16(2000 + dist, 0, n, dist)
        es = oracle.exact_sum_bf16(bits)
        for off in (0, 3):
            g, g64 = _sum(tcr, _dev(bits, off), algo)
            assert oracle.within_tolerance(g, es), (algo, dist, n, off, g, es.f64())
            assert oracle.within_tolerance(g64, es)
        if dist == gen.ONES:
            assert g == float(n)


@pytest.mark.parametrize("algo", ALGOS)
def test_bf16_integers_bitwise(tcr, algo):
    bits = gen.generate_bf16(8, 0, (1 << 21) + 17, gen.SMALLINT)
    es = oracle.exact_sum_bf16(bits)
    assert _sum(tcr, _dev(bits, 1), algo)[0] == float(es.value)


def test_bf16_full_size_c3(tcr):
    import torch

    n = 1 << 30
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1, bf16=True)
    bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    es = oracle.ExactSum(0, 0, unit_exp=-133)
    for lo in range(0, n, 1 << 26):
        es = es + oracle.exact_sum_bf16(bits[lo:lo + (1 << 26)])
    for algo in ("default",) + tuple(ALGOS):
        g, _ = _sum(tcr, x, algo)
        assert oracle.within_tolerance(g, es), (algo, g, es.f64())


@pytest.mark.parametrize("algo", ["mma_sync", "shuffle"])
def test_bf16_segmented(tcr, algo):
    import torch

    lens = gen.loguniform_lengths(77, 3000)
    off = gen.offsets_from_lengths(lens, start=3)
    bits = gen.generate_bf16(77, 0, int(off[-1]) + 5, gen.WIDE)
    out = torch.empty(3000, dtype=torch.float32, device="cuda")
    tcr.tcr_reduce_sum_segmented_ex(_dev(bits, 1), torch.from_numpy(off).cuda(), out, algo=algo)
    torch.cuda.synchronize()
    g = out.cpu().numpy()
    for j in range(0, 3000, 7):
        es = oracle.exact_sum_bf16(bits[off[j]:off[j + 1]])
        assert oracle.within_tolerance(float(g[j]), es), (j, g[j], es.f64())


def test_ex_rejects_unknown_dtype(tcr):
    import torch

    x = torch.zeros(16, dtype=torch.float16, device="cuda")
    o = torch.empty(1, dtype=torch.float32, device="cuda")
    with pytest.raises(tcr.TcrError):
        tcr.tcr_reduce_sum_ex(x, out_f32=o, dtype=7)


def _bdev(bits, off=0):
    import torch

    buf = torch.zeros(bits.size + off + 16, dtype=torch.int16, device="cuda")
    x = buf[off:off + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits.view(np.int16)))
    return x.view(torch.bfloat16)


def _exact_bf16(tcr, x):
    import torch

    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    o64 = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    tcr.tcr_reduce_sum_exact_ex(x, out_f32=o32, out_f64=o64)
    torch.cuda.synchronize()
    return float(o32.item()), float(o64.item())


@pytest.mark.parametrize("n", [0, 1, 7, 255, 256, 257, 4097, 100_003, 3_000_017])
def test_bf16_exact_bitwise(tcr, n):
    """NEXT-3 x NEXT-4: exact bfloat16 (8 exponent windows) is bitwise equal to
    the exact bf16 oracle (per-exponent bins), every distribution, misaligned."""
    for dist in (gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01, gen.SMALLINT, gen.ONES):
        bits = gen.generate_bf16(n + dist, 0, n, dist)
        es = oracle.exact_sum_bf16(bits)
        for off in ((0, 1, 5) if n < 5000 else (3,)):
            g32, g64 = _exact_bf16(tcr, _bdev(bits, off))
            assert g32 == es.f32() and g64 == es.f64(), (n, dist, off, g32, g64, es.f64())


def test_bf16_exact_extreme_ranges(tcr):
    """Values from every exponent window at once, subnormals, cancellation of
    huge values leaving tiny ones, overflow past binary32, and all finite
    bf16 patterns (their sum is exactly 0)."""
    rng = np.random.default_rng(11)
    cases = []
    for _ in range(20):  # random patterns over the whole finite range
        h = rng.integers(0, 1 << 16, 50_000).astype(np.uint16)
        h = h[((h >> 7) & 0xFF) != 0xFF]
        cases.append(h)
    big, tiny = 0x7F7F, 0x0001  # max finite, min subnormal
    cases.append(np.array([big, big ^ 0x8000, tiny] * 1000, dtype=np.uint16))  # -> 1000 * 2^-133
    cases.append(np.array([big] * 10, dtype=np.uint16))  # overflows binary32 -> inf
    cases.append(np.array([h for h in range(1 << 16) if ((h >> 7) & 0xFF) != 0xFF], dtype=np.uint16))
    for i, bits in enumerate(cases):
        es = oracle.exact_sum_bf16(bits)
        g32, g64 = _exact_bf16(tcr, _bdev(bits, i % 3))
        assert g32 == es.f32() and g64 == es.f64(), (i, g32, g64, es.f64())


def test_bf16_exact_specials(tcr):
    import math

    bits = gen.generate_bf16(1, 0, 10_000, gen.UNIFORM_PM1)
    for special, kind in ((0x7F80, "+inf"), (0xFF80, "-inf"), (0x7FC1, "nan")):
        b = bits.copy()
        b[4321] = special
        g32, g64 = _exact_bf16(tcr, _bdev(b))
        if kind == "nan":
            assert math.isnan(g32) and math.isnan(g64)
        else:
            assert g32 == g64 == (math.inf if kind == "+inf" else -math.inf)
    b = bits.copy()
    b[10], b[20] = 0x7F80, 0xFF80
    g32, _ = _exact_bf16(tcr, _bdev(b))
    assert math.isnan(g32)
