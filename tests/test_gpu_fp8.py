"""NEXT-4: fp8 (E4M3 / E5M2) inputs through the MMA encoding (mma.sync
m16n8k32 and tcgen05 kind::f8f6f4, B = fp8 ones) and the shuffle path, vs the
exact fp8 oracle; tolerance |g - R| <= 2^-20 * sum|x_i|; any byte alignment."""
import numpy as np
import pytest

import oracle
import tcr_inputs as gen

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
