"""tcgen05 dynamic tail (TCR_CFG_TC05_DYNAMIC, r02).

Each CTA streams its own contiguous run of the first (100 - d) % of the
chunks, then takes the remaining chunks one at a time from a counter.  The
rounds are combined exactly (integer units of 2^-24 after the per-round DMMA
collapse), so WHICH CTA reduced a chunk cannot change the result: every
d > 0 must give the same bits, for every size, alignment, format and ring
shape; and the result must satisfy the north-star tolerance against the
exact oracle (Eq. 2).  Expected values come only from oracle/.
"""
import contextlib
import os

import numpy as np
import pytest

import oracle
import tcr_inputs as gen

pytestmark = pytest.mark.gpu

DYNS = [1, 25, 50, 100]


@pytest.fixture(scope="module")
def tcr():
    import torch

    torch.cuda.set_device(0)
    import paper_1903_03640_b200 as m

    return m


@contextlib.contextmanager
def _cfg(tcr, **kv):
    keys = {k: getattr(tcr, "TCR_CFG_" + k.upper()) for k in kv}
    saved = {k: tcr.tcr_get_config(v) for k, v in keys.items()}
    try:
        for k, v in kv.items():
            tcr.tcr_set_config(keys[k], v)
        yield
    finally:
        for k, v in saved.items():
            tcr.tcr_set_config(keys[k], v)


def _dev16(bits, offset=0):
    import torch

    buf = torch.empty(bits.size + offset + 8, dtype=torch.int16, device="cuda")
    x = buf[offset:offset + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits.view(np.int16)))
    return x.view(torch.float16)


def _sum(tcr, x, f64=False):
    import torch

    o32 = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    o64 = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    tcr.tcr_reduce_sum_ex(x, out_f32=o32, out_f64=o64, algo="tcgen05")
    torch.cuda.synchronize()
    return (float(o32.item()), float(o64.item())) if f64 else float(o32.item())


def _bits32(v):
    return np.float32(v).view(np.uint32)


@pytest.fixture(autouse=True)
def _dyn_at_every_size(tcr):
    """The library keeps short inputs (static runs < 32 chunks per CTA) on the
    static partition; the tests below take the dynamic tail at every size."""
    with _cfg(tcr, tc05_dyn_min_run=0):
        yield


def test_knob_defaults_and_range(tcr):
    assert tcr.tcr_get_config(tcr.TCR_CFG_TC05_DYNAMIC) == 8
    for key, bad in ((tcr.TCR_CFG_TC05_DYNAMIC, -1), (tcr.TCR_CFG_TC05_DYNAMIC, 101),
                     (tcr.TCR_CFG_TC05_DYN_MIN_RUN, -1)):
        with pytest.raises(tcr.TcrError):
            tcr.tcr_set_config(key, bad)
    assert tcr.tcr_get_config(tcr.TCR_CFG_TC05_DYNAMIC) == 8


def test_default_min_run_gate(tcr):
    """With the default gate (32 chunks per CTA) a short input takes the static
    partition and a long one the dynamic tail; both within tolerance, and the
    long one bitwise equal to an explicit d = 8, min-run 0 call."""
    for n in ((1 << 22) + 3, (1 << 28) + 16384 * 3 + 5):
        bits = gen.generate(4242, 0, n, gen.UNIFORM_PM1)
        es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
        x = _dev16(bits, 1)
        with _cfg(tcr, tc05_dyn_min_run=32):
            g = _sum(tcr, x)
        with _cfg(tcr, tc05_dynamic=0):
            g0 = _sum(tcr, x)
        with _cfg(tcr, tc05_dynamic=50):
            g50 = _sum(tcr, x)
        assert oracle.within_tolerance(g, es), (n, g, es.f64())
        assert _bits32(g) == _bits32(g0) == _bits32(g50), (n, g, g0, g50)


# sizes: below one 32 KiB stage (ragged only), one stage +- 1, a few stages
# with a ragged tail, fewer chunks than CTAs, and many chunks per CTA (the
# 1-CTA/SM shape starts at 256 MiB: 2^27 elements)
SIZES = [1, 16383, 16384, 16385, 5 * 16384 + 333, 148 * 16384 - 1, (1 << 22) + 123,
         3 * (1 << 20) + 4099, (1 << 26) + 5, (1 << 27) + 16384 * 7 + 19]


@pytest.mark.parametrize("n", SIZES)
def test_schedule_invariance_binary16(tcr, n):
    bits = gen.generate(1603 + n % 97, 0, n, gen.UNIFORM_PM1)
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
    for off in (0, 3):
        x = _dev16(bits, off)
        got = {}
        for d in [0] + DYNS:
            with _cfg(tcr, tc05_dynamic=d):
                got[d] = _sum(tcr, x, f64=True)
        for d, (g, g64) in got.items():
            assert oracle.within_tolerance(g, es), (n, off, d, g, es.f64())
            assert oracle.within_tolerance(g64, es), (n, off, d, g64)
        ref = got[DYNS[0]]
        for d in DYNS[1:]:
            assert _bits32(got[d][0]) == _bits32(ref[0]) and got[d][1] == ref[1], (n, off, d, got)
        # uniform[-1, 1]: the static path's binary64 additions are exact too
        # (|partial sums| << 2^29), so it agrees bit for bit
        assert got[0] == ref, (n, off, got)


@pytest.mark.parametrize("dist", [gen.UNIFORM_01, gen.WIDE, gen.ALTERNATING, gen.ONES, gen.SMALLINT])
def test_schedule_invariance_distributions(tcr, dist):
    n = (1 << 24) + 16384 * 3 + 77
    bits = gen.generate(2207 + dist, 0, n, dist)
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
    x = _dev16(bits, 1)
    got = {}
    for d in DYNS:
        with _cfg(tcr, tc05_dynamic=d):
            got[d] = _sum(tcr, x, f64=True)
    for d, (g, g64) in got.items():
        assert oracle.within_tolerance(g, es), (dist, d, g, es.f64())
    assert len({(_bits32(g), g64) for g, g64 in got.values()}) == 1, (dist, got)
    if dist in (gen.ONES, gen.SMALLINT):  # every fp32 row sum exact: the result is RNE(R(X))
        assert got[25][0] == es.f32() and got[25][1] == es.f64(), (dist, got[25], es.value)


def test_exact_combination_of_large_sums(tcr):
    """Whole 32 KiB chunks of 65504 and, every 16th chunk, of the smallest
    subnormal 2^-24: every fp32 row sum is exact (a row never mixes the two),
    the total ~2^43 needs 2^-10 resolution (54 bits), and the integer combine
    returns RNE53 / RNE24 of R(X) (Eq. 2) exactly, for any schedule."""
    n = (1 << 27) + 16384 * 5
    bits = np.full(n, 0x7BFF, dtype=np.uint16)  # 65504
    bits.reshape(-1, 16384)[::16] = 0x0001       # 2^-24
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
    x = _dev16(bits)
    for d in (25, 100):
        with _cfg(tcr, tc05_dynamic=d):
            g, g64 = _sum(tcr, x, f64=True)
        assert g == es.f32() and g64 == es.f64(), (d, g, g64, es.f32(), es.f64())


@pytest.mark.parametrize("fmt", [oracle.FP8_E4M3, oracle.FP8_E5M2])
def test_schedule_invariance_fp8(tcr, fmt):
    import torch

    for n in (17, 32768 * 5 + 9, (1 << 23) + 333, (1 << 28) + 32768 * 3 + 1):
        bits = gen.generate_fp8(51, 0, n, gen.WIDE, fmt)
        es = oracle.exact_sum_fp8(bits, fmt)
        buf = torch.empty(n + 24, dtype=torch.uint8, device="cuda")
        x = buf[5:5 + n]
        x.copy_(torch.from_numpy(bits))
        x = x.view(torch.float8_e4m3fn if fmt == oracle.FP8_E4M3 else torch.float8_e5m2)
        got = {}
        for d in [0] + DYNS:
            with _cfg(tcr, tc05_dynamic=d):
                got[d] = _sum(tcr, x)
        for d, g in got.items():
            assert oracle.within_tolerance(g, es), (fmt, n, d, g, es.f64())
        assert len({_bits32(got[d]) for d in DYNS}) == 1, (fmt, n, got)


def test_specials_in_static_and_dynamic_chunks(tcr):
    n = (1 << 24) + 999
    base = gen.generate(9, 0, n, gen.UNIFORM_PM1)
    for d in (25, 100):
        with _cfg(tcr, tc05_dynamic=d):
            for pos in (0, 12345, n // 2, n - 20000, n - 5):  # static runs, dynamic tail, ragged end
                bits = base.copy()
                bits[pos] = 0x7C00  # +inf
                assert _sum(tcr, _dev16(bits)) == float("inf"), (d, pos)
                bits[pos] = 0xFC00  # -inf
                assert _sum(tcr, _dev16(bits)) == float("-inf"), (d, pos)
                bits[pos] = 0x7E00  # NaN
                g = _sum(tcr, _dev16(bits))
                assert g != g, (d, pos)
            bits = base.copy()
            bits[100] = 0x7C00
            bits[n - 100] = 0xFC00  # +inf and -inf -> NaN
            g = _sum(tcr, _dev16(bits))
            assert g != g, d


@pytest.mark.parametrize("shape", [(4, 16, 4, 1, 1), (4, 32, 4, 2, 1), (3, 64, 4, 4, 1),
                                   (2, 32, 4, 2, 3), (4, 32, 4, 2, 2), (8, 16, 4, 1, 1)])
def test_ring_shapes(tcr, shape):
    """4, 8 and 16 MMAs per stage, 1-3 CTAs per SM: each shape schedule-invariant."""
    st, kb, sl, ch, ct = shape
    n = (1 << 25) + 4097
    bits = gen.generate(77, 0, n, gen.UNIFORM_01)
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
    x = _dev16(bits, 2)
    with _cfg(tcr, tc05_stages=st, tc05_stage_kb=kb, tc05_slots=sl, tc05_chain=ch,
              tc05_ctas_per_sm=ct):
        got = {}
        for d in DYNS:
            with _cfg(tcr, tc05_dynamic=d):
                got[d] = _sum(tcr, x)
    for d, g in got.items():
        assert oracle.within_tolerance(g, es), (shape, d, g, es.f64())
    assert len({_bits32(g) for g in got.values()}) == 1, (shape, got)


def test_counter_resets_between_launches(tcr):
    """The chunk counter self-resets: 60 launches interleaving sizes, algorithms
    and PDL on / off on one stream give the bits of the first call each time."""
    import torch

    xs = [_dev16(gen.generate(s, 0, n, gen.UNIFORM_PM1), s % 4)
          for s, n in ((1, (1 << 22) + 7), (2, (1 << 20) + 5), (3, 16385))]
    first = [_sum(tcr, x) for x in xs]
    for i in range(60):
        with _cfg(tcr, pdl=i % 2):
            j = i % 3
            o = torch.empty(1, dtype=torch.float32, device="cuda")
            if i % 5 == 0:
                tcr.tcr_reduce_sum_algo(xs[j], out_f32=o, algo="mma_sync")
            g = _sum(tcr, xs[j])
            assert _bits32(g) == _bits32(first[j]), (i, j, g, first[j])


def test_cuda_graph_replay(tcr):
    import torch

    x = _dev16(gen.generate(8, 0, (1 << 23) + 3, gen.UNIFORM_PM1))
    want = _sum(tcr, x)
    o = torch.empty(1, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="tcgen05", stream=s)  # workspace for s
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                tcr.tcr_reduce_sum_algo(x, out_f32=o, algo="tcgen05", stream=s)
    for _ in range(4):
        o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert _bits32(o.item()) == _bits32(want)


def test_full_size_c3(tcr):
    """BASELINE config 3 (2^30 binary16): every d > 0 gives the same bits, within
    the tolerance of the exact sum."""
    import torch

    n = 1 << 30
    x = gen.generate_tensor(gen.SEED_C3, 0, n, gen.UNIFORM_PM1)
    bits = x.view(torch.int16).cpu().numpy().view(np.uint16)
    es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 8)
    got = {}
    for d in (0, 10, 25, 100):
        with _cfg(tcr, tc05_dynamic=d):
            got[d] = _sum(tcr, x, f64=True)
    for d, (g, g64) in got.items():
        assert oracle.within_tolerance(g, es), (d, g, es.f64())
    assert got[10] == got[25] == got[100], got


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_fused_peer_combine_emulated(tcr, P):
    """NEXT-2 on the dynamic-tail kernel: P emulated ranks (one cooperative
    launch, a chunk counter and 3-word partials per rank slice) -- every rank
    returns the same total, within tolerance, and equal to the plain kernel's
    total for P = 1; integer data exact."""
    import torch

    boxes = [tcr.tcr_peer_mailbox_alloc() for _ in range(P)]
    try:
        n = (1 << 24) + 16384 * 5 + 3
        o32 = torch.full((P,), float("nan"), dtype=torch.float32, device="cuda")
        o64 = torch.full((P,), float("nan"), dtype=torch.float64, device="cuda")
        for epoch, dist in enumerate((gen.UNIFORM_PM1, gen.WIDE, gen.SMALLINT)):
            bits = gen.generate(60 + epoch, 0, n, dist)
            x = _dev16(bits)
            es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
            for d in (0, 8, 100):
                with _cfg(tcr, tc05_dynamic=d):
                    tcr.tcr_reduce_sum_peer_emulated(x, boxes, out_f32=o32, out_f64=o64, algo="tcgen05")
                    torch.cuda.synchronize()
                    g32, g64 = o32.cpu().tolist(), o64.cpu().tolist()
                    assert len(set(g64)) == 1 and len(set(g32)) == 1, (P, d, epoch, g64)
                    assert oracle.within_tolerance(g32[0], es), (P, d, epoch, g32[0], es.f64())
                    if dist == gen.SMALLINT:
                        assert g64[0] == es.f64() and g32[0] == es.f32(), (P, d, g64[0])
                    if P == 1:
                        assert g32[0] == _sum(tcr, x), (d, epoch)
        for b in boxes:
            assert not tcr.tcr_peer_mailbox_error(b)
    finally:
        torch.cuda.synchronize()
        for b in boxes:
            tcr.tcr_peer_mailbox_free(b)


def test_e4m3_default_path_is_exact(tcr):
    """fp8 E4M3 values are multiples of 2^-9 below 448: a row of the default
    stage (2 MMAs x 32 elements = 64 values) sums to < 2^24 units of 2^-9, so
    every binary32 row sum is exact, the per-round D' = 1 x D collapse is
    exact and the integer combine is exact -- the default large-n E4M3 path
    returns RNE(R(X)) bit for bit (binary32 and binary64), for any schedule."""
    import torch

    n = (1 << 29) + 32768 * 3 + 17  # >= 512 MiB: the tcgen05 dynamic-tail default
    assert tcr.tcr_default_algo(n, tcr.TCR_DTYPE_E4M3) == tcr.TCR_ALGO_TCGEN05
    for dist in (gen.UNIFORM_PM1, gen.WIDE):
        x = gen.generate_tensor_fp8(90 + dist, 0, n, dist, gen.FP8_E4M3)
        bits = x.view(torch.uint8).cpu().numpy()
        es = oracle.exact_sum_fp8(bits, oracle.FP8_E4M3)
        o32 = torch.empty(1, dtype=torch.float32, device="cuda")
        o64 = torch.empty(1, dtype=torch.float64, device="cuda")
        for d in (8, 100):
            with _cfg(tcr, tc05_dynamic=d, tc05_dyn_min_run=32):
                tcr.tcr_reduce_sum_ex(x, out_f32=o32, out_f64=o64)
                torch.cuda.synchronize()
            assert o32.item() == es.f32() and o64.item() == es.f64(), (dist, d, o64.item(), es.f64())


def test_e4m3_exact_adversarial_rows(tcr):
    """The sharpest case for the claim above: every element 448 (the E4M3
    maximum) except one smallest subnormal 2^-9 per 4 KiB -- the rows holding
    it sum 63 x 448 + 2^-9, which needs all 24 bits of a binary32.  The
    binary64 result resolves the 2^-9 terms (~2^38 total, ulp 2^-15)."""
    import torch

    n = 1 << 29
    bits = np.full(n, 0x7E, dtype=np.uint8)  # 448
    bits[::4096] = 0x01                      # 2^-9
    bits[2048::4096] = 0xFE                  # -448: keeps the total's ulp small enough
    es = oracle.exact_sum_fp8(bits, oracle.FP8_E4M3)
    x = torch.from_numpy(bits).cuda().view(torch.float8_e4m3fn)
    o32 = torch.empty(1, dtype=torch.float32, device="cuda")
    o64 = torch.empty(1, dtype=torch.float64, device="cuda")
    tcr.tcr_reduce_sum_ex(x, out_f32=o32, out_f64=o64)
    torch.cuda.synchronize()
    assert o64.item() == es.f64() and o32.item() == es.f32(), (o64.item(), es.f64())


def test_random_fuzz_flat(tcr):
    """30 random flat problems on the dynamic-tail kernel (binary16 and fp8):
    random size up to 2^25, byte offset, distribution, dynamic fraction and
    ring shape (4 / 8 / 16 MMAs per stage) -- within tolerance of the exact
    oracle and bitwise equal across two dynamic fractions."""
    import torch

    rng = np.random.default_rng(1903)
    shapes = [(4, 16, 4, 1), (4, 32, 4, 2), (3, 64, 4, 4)]
    for it in range(30):
        f8 = it % 3 == 2
        n = int(rng.integers(1, 1 << 25))
        dist = int(rng.choice([gen.UNIFORM_PM1, gen.WIDE, gen.UNIFORM_01, gen.ALTERNATING]))
        st, kb, sl, ch = shapes[int(rng.integers(0, 3 if not f8 else 2))]
        d1, d2 = (int(v) for v in rng.choice([1, 8, 25, 60, 100], size=2, replace=False))
        if f8:
            fmt = oracle.FP8_E4M3 if it % 2 else oracle.FP8_E5M2
            bits = gen.generate_fp8(it, 0, n, dist, fmt)
            es = oracle.exact_sum_fp8(bits, fmt)
            off = int(rng.integers(0, 16))
            buf = torch.empty(n + 32, dtype=torch.uint8, device="cuda")
            x = buf[off:off + n]
            x.copy_(torch.from_numpy(bits))
            x = x.view(torch.float8_e4m3fn if fmt == oracle.FP8_E4M3 else torch.float8_e5m2)
        else:
            bits = gen.generate(it, 0, n, dist)
            es = oracle.exact_sum_fp16(bits, threads=os.cpu_count() or 4)
            x = _dev16(bits, int(rng.integers(0, 8)))
        with _cfg(tcr, tc05_stages=st, tc05_stage_kb=kb, tc05_slots=sl, tc05_chain=ch):
            with _cfg(tcr, tc05_dynamic=d1):
                g1 = _sum(tcr, x)
            with _cfg(tcr, tc05_dynamic=d2):
                g2 = _sum(tcr, x)
        assert oracle.within_tolerance(g1, es), (it, n, f8, dist, g1, es.f64())
        assert _bits32(g1) == _bits32(g2), (it, n, f8, d1, d2, g1, g2)
