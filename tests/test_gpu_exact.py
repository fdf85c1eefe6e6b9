"""NEXT-3: the exact GPU reduction must equal the exact oracle BIT FOR BIT
(integer T in units of 2^-24, and the correctly rounded binary32/binary64),
for every input, size, alignment and shard count."""
import os

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


def _dev(bits, offset=0):
    import torch

    buf = torch.empty(bits.size + offset + 8, dtype=torch.int16, device="cuda")
    x = buf[offset:offset + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits.view(np.int16)))
    return x.view(torch.float16)


def _exact(tcr, x):
    import torch

    acc = torch.full((6,), -7, dtype=torch.int64, device="cuda")
    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    o64 = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    tcr.tcr_reduce_sum_exact(x, acc=acc, out_f32=o32, out_f64=o64)
    torch.cuda.synchronize()
    a = acc.cpu().tolist()
    return a, float(o32.item()), float(o64.item())


def _check(tcr, a, g32, g64, es):
    assert exact_limbs_to_int(a) == es.T
    assert 0 <= a[0] < (1 << 40) and 0 <= a[1] < (1 << 40)
    assert (a[3], a[4], a[5]) == (es.n_nan, es.n_pinf, es.n_ninf)
    r32, r64 = es.f32(), es.f64()
    if r32 != r32:
        assert g32 != g32 and g64 != g64
    else:
        assert g32 == r32 and g64 == r64, (g32, r32, g64, r64)
        assert np.signbit(g32) == np.signbit(np.float32(r32)) or g32 != 0.0


SIZES = [0, 1, 2, 7, 8, 9, 255, 256, 257, 8191, 65536 + 37, (1 << 20) + 5, 3 * (1 << 21) + 4099]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", [gen.UNIFORM_PM1, gen.UNIFORM_01, gen.WIDE, gen.ALTERNATING])
def test_exact_bitwise(tcr, n, dist):
    bits = gen.generate(4242 + dist, 0, n, dist)
    es = oracle.exact_sum_fp16(bits)
    for off in (0, 5):
        _check(tcr, *_exact(tcr, _dev(bits, off)), es)


def test_exact_extremes_and_specials(tcr):
    # max-magnitude values: |T| far beyond 2^64 units; subnormals; ties in the final rounding
    cases = [
        np.full(3_000_001, np.float16(65504.0)).view(np.uint16),
        np.full(1_000_000, np.float16(-65504.0)).view(np.uint16),
        np.arange(1, 1024, dtype=np.uint16),                       # subnormals only
        np.array([0x3C00, 0x0001], dtype=np.uint16),               # 1 + 2^-24: a binary32 tie
        np.array([0x3C00, 0x0001, 0x0001], dtype=np.uint16),       # 1 + 2^-23
        np.array([0x3C00, 0x0003], dtype=np.uint16),               # 1 + 3*2^-24: rounds up
        np.array([0x8000, 0x0000], dtype=np.uint16),               # -0 + 0
    ]
    for bits in cases:
        es = oracle.exact_sum_fp16(bits)
        _check(tcr, *_exact(tcr, _dev(bits, 1)), es)
    bits = gen.generate(3, 0, 100_000, gen.UNIFORM_PM1)
    for pos, val in ((10, 0x7C00), (20, 0xFC00), (30, 0x7E01)):
        b2 = bits.copy()
        b2[pos] = val
        es = oracle.exact_sum_fp16(b2)
        _check(tcr, *_exact(tcr, _dev(b2)), es)
    b2 = bits.copy()
    b2[5], b2[6] = 0x7C00, 0xFC00
    _check(tcr, *_exact(tcr, _dev(b2)), oracle.exact_sum_fp16(b2))


def test_exact_full_size_c3(tcr):
    import torch

    n = 1 << 30
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 8)
    _check(tcr, *_exact(tcr, x), es)
    assert _exact(tcr, x) == _exact(tcr, x)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_exact_sharded_is_independent_of_P(tcr, P):
    """Per-shard exact accumulators summed as int64 (what an NCCL SUM allreduce
    does) and finalized give the same bits as the single-GPU result."""
    import torch

    n = (1 << 24) + 333
    bits = gen.generate(gen.SEED_C4, 0, n, gen.UNIFORM_01)
    es = oracle.exact_sum_fp16(bits, threads=8)
    x = _dev(bits)
    accs = torch.empty((P, 6), dtype=torch.int64, device="cuda")
    for r in range(P):
        lo, hi = r * n // P, (r + 1) * n // P
        tcr.tcr_reduce_sum_exact(x[lo:hi], acc=accs[r])
    tot = accs.sum(dim=0)  # the allreduce
    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    tcr.tcr_exact_finalize(tot, out_f32=o32, out_f64=o64)
    torch.cuda.synchronize()
    t = tot.cpu().tolist()
    assert exact_limbs_to_int(t) == es.T
    assert float(o32.item()) == es.f32() and float(o64.item()) == es.f64()


@pytest.mark.parametrize("n", [1, 9, 16384 * 2 + 7, (1 << 20) + 5, 3 * (1 << 21) + 4099, (1 << 27) + 16384 * 3 + 11])
def test_exact_bulk_kernel_bitwise(tcr, n):
    """The TMA-fed exact kernel with the dynamic tail (TCR_CFG_EXACT_BULK = 2
    forces it at every size; r02 §18) equals the oracle bit for bit, for
    static and dynamic chunk schedules, aligned and misaligned, with specials
    in static runs, dynamic chunks and the ragged end."""
    keys = (tcr.TCR_CFG_EXACT_BULK, tcr.TCR_CFG_TC05_DYNAMIC, tcr.TCR_CFG_TC05_DYN_MIN_RUN)
    saved = [tcr.tcr_get_config(k) for k in keys]
    try:
        tcr.tcr_set_config(tcr.TCR_CFG_EXACT_BULK, 2)
        tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYN_MIN_RUN, 0)
        for dist in (gen.UNIFORM_PM1, gen.WIDE):
            bits = gen.generate(8800 + dist, 0, n, dist)
            es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
            for d in (0, 8, 100):
                tcr.tcr_set_config(tcr.TCR_CFG_TC05_DYNAMIC, d)
                for off in (0, 3):
                    _check(tcr, *_exact(tcr, _dev(bits, off)), es)
        if n > 100:
            for pos in (0, n // 2, n - 3):
                b2 = gen.generate(5, 0, n, gen.UNIFORM_PM1)
                b2[pos] = 0x7C00
                _check(tcr, *_exact(tcr, _dev(b2, 1)), oracle.exact_sum_fp16(b2))
    finally:
        for k, v in zip(keys, saved):
            tcr.tcr_set_config(k, v)
