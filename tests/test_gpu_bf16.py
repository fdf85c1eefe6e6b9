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
