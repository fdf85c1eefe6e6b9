"""GPU parity of the segmented / batched entry points (BASELINE config 5),
and of the device input generator against its host definition."""
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

    return m


def _dev(bits, offset=0):
    import torch

    buf = torch.empty(bits.size + offset + 8, dtype=torch.int16, device="cuda")
    x = buf[offset:offset + bits.size]
    x.copy_(torch.from_numpy(bits.view(np.int16)))
    return x.view(torch.float16)


def _seg(tcr, x, off, mma=True):
    import torch

    out = torch.full((len(off) - 1,), float("nan"), dtype=torch.float32, device="cuda")
    f = tcr.tcr_reduce_sum_segmented if mma else tcr.tcr_reduce_sum_segmented_shuffle
    f(x, torch.from_numpy(np.asarray(off, dtype=np.int64)).cuda(), out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("mma", [True, False])
def test_generator_device_matches_host(tcr, mma):
    import torch

    for dist in range(6):
        for start, n in ((0, 1), (5, 1000), (1 << 33, 100_003)):
            d = gen.generate_tensor(17 + dist, start, n, dist).view(torch.int16).cpu().numpy()
            assert np.array_equal(d.view(np.uint16), gen.generate(17 + dist, start, n, dist)), dist


@pytest.mark.parametrize("mma", [True, False])
def test_edge_segments(tcr, mma):
    n = 300_000
    bits = gen.generate(12, 0, n, gen.UNIFORM_PM1)
    lens = [0, 1, 2, 7, 8, 9, 15, 16, 17, 255, 256, 257, 0, 4095, 4096, 4097, 65536, 0, 1, 33333]
    starts = [0, 3, 11, 100, 1001]
    for s0 in starts:
        off = gen.offsets_from_lengths(np.array(lens), start=s0)
        assert off[-1] <= n
        for xoff in (0, 3):
            g = _seg(tcr, _dev(bits, xoff), off, mma)
            ref = oracle.exact_segment_sums_fp16(bits, off)
            for j, (gj, rj) in enumerate(zip(g.tolist(), ref)):
                assert oracle.within_tolerance(gj, rj), (mma, s0, xoff, j, gj, rj.f64())
                if lens[j] == 0:
                    assert gj == 0.0


@pytest.mark.parametrize("mma", [True, False])
def test_segment_index_bit_exact(tcr, mma):
    # All-ones data and pairwise-distinct lengths: out[j] must equal len(j)
    # exactly, so any permutation or off-by-one of the output index fails.
    rng = np.random.default_rng(0)
    lens = rng.permutation(np.arange(0, 6000, 3))
    off = gen.offsets_from_lengths(lens, start=5)
    bits = np.full(int(off[-1]) + 8, 0x3C00, dtype=np.uint16)
    g = _seg(tcr, _dev(bits, 1), off, mma)
    assert np.array_equal(g, lens.astype(np.float32))


@pytest.mark.parametrize("mma", [True, False])
def test_loguniform_mix(tcr, mma):
    S = 4096
    lens = gen.loguniform_lengths(gen.SEED_C5, S)
    off = gen.offsets_from_lengths(lens)
    n = int(off[-1])
    for dist in (gen.UNIFORM_PM1, gen.UNIFORM_01, gen.WIDE):
        bits = gen.generate(gen.SEED_C5, 0, n, dist)
        g = _seg(tcr, _dev(bits), off, mma)
        ref = oracle.exact_segment_sums_fp16(bits, off)
        bad = [j for j in range(S) if not oracle.within_tolerance(float(g[j]), ref[j])]
        assert not bad, (dist, bad[:5])
        # deterministic across runs
        assert np.array_equal(g, _seg(tcr, _dev(bits), off, mma))


@pytest.mark.parametrize("mma", [True, False])
def test_batched(tcr, mma):
    import torch

    # aligned x with L in {256, 512, 1024, 2048} takes the whole-tile rows kernel
    cases = ((1, 1000), (7, 333), (256, 4096), (256, 4093), (512, 999), (1000, 777),
             (1024, 1025), (2048, 33), (4096, 1024), (65536, 17))
    for L, S in cases:
        bits = gen.generate(L, 0, L * S, gen.UNIFORM_PM1)
        ref = oracle.exact_segment_sums_fp16(bits, np.arange(S + 1, dtype=np.int64) * L)
        for xoff in (0, 2):
            x = _dev(bits, xoff)
            out = torch.full((S,), float("nan"), dtype=torch.float32, device="cuda")
            f = tcr.tcr_reduce_sum_batched if mma else tcr.tcr_reduce_sum_batched_shuffle
            f(x, L, out)
            torch.cuda.synchronize()
            g = out.cpu().numpy()
            assert all(oracle.within_tolerance(float(g[j]), ref[j]) for j in range(S)), (L, S, xoff)


def test_empty_and_zero_segments(tcr):
    import torch

    out = torch.empty(0, dtype=torch.float32, device="cuda")
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    x = torch.empty(0, dtype=torch.float16, device="cuda")
    tcr.tcr_reduce_sum_segmented(x, off, out, num_segments=0)
    torch.cuda.synchronize()


@pytest.mark.parametrize("mma", [True, False])
def test_random_fuzz_against_oracle(tcr, mma):
    """200 random CSR problems: random segment counts (0..300), length mixes
    (empty, short, tile-crossing, long), start offsets, x misalignment and
    distributions; every segment vs the exact oracle, empty ones exactly 0,
    and a second launch bitwise identical."""
    import torch

    rng = np.random.default_rng(2024 + mma)
    for case in range(200):
        S = int(rng.integers(0, 300))
        kind = rng.integers(0, 4, S)
        lens = np.where(kind == 0, 0, np.where(kind == 1, rng.integers(1, 40, S),
                        np.where(kind == 2, rng.integers(200, 600, S), rng.integers(1000, 20000, S))))
        start = int(rng.integers(0, 50))
        off = gen.offsets_from_lengths(lens.astype(np.int64), start=start)
        dist = int(rng.choice([gen.UNIFORM_PM1, gen.UNIFORM_01, gen.WIDE, gen.SMALLINT]))
        bits = gen.generate(case, 0, int(off[-1]) + 9, dist)
        xoff = int(rng.integers(0, 8))
        x = _dev(bits, xoff)
        if S == 0:
            out = torch.empty(0, dtype=torch.float32, device="cuda")
            f = tcr.tcr_reduce_sum_segmented if mma else tcr.tcr_reduce_sum_segmented_shuffle
            f(x, torch.from_numpy(off).cuda(), out, num_segments=0)
            continue
        g = _seg(tcr, x, off, mma)
        ref = oracle.exact_segment_sums_fp16(bits, off)
        for j in range(S):
            assert oracle.within_tolerance(float(g[j]), ref[j]), (case, j, g[j], ref[j].f64())
            if lens[j] == 0:
                assert g[j] == 0.0
            if dist == gen.SMALLINT:
                assert float(g[j]) == ref[j].f32()
        assert np.array_equal(g, _seg(tcr, x, off, mma)), case
