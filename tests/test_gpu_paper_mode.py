"""The paper's algorithm taken literally (study mode, tcr_reduce_sum_paper_f16):
fp16 MMAs, fp16 partials written to memory, one launch per level."""
import math

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


def _run(tcr, bits, offset=0):
    import torch

    buf = torch.zeros(bits.size + offset + 16, dtype=torch.int16, device="cuda")
    x = buf[offset:offset + bits.size]
    if bits.size:
        x.copy_(torch.from_numpy(bits.view(np.int16)))
    out = torch.full((1,), float("nan"), dtype=torch.float32, device="cuda")
    l0 = tcr.tcr_launch_count()
    tcr.tcr_reduce_sum_paper_f16(x.view(torch.float16), out)
    torch.cuda.synchronize()
    return float(out.item()), tcr.tcr_launch_count() - l0


def _levels(n):  # ceil(log_256 n), at least one level for n >= 1 (Eq. 13-14)
    lv, m = 0, n
    while True:
        m = (m + 255) // 256
        lv += 1
        if m <= 1:
            return lv


@pytest.mark.parametrize("n", [1, 7, 255, 256, 257, 2048, 4097, 32768, 1 << 20])
def test_ones_exact_and_one_launch_per_level(tcr, n):
    """All-ones: every group partial is an integer <= 256 (exact in binary16);
    the level above adds them in binary16, so the result is n rounded to
    binary16 (4097 -> 4096); one launch per level."""
    bits = gen.generate(0, 0, n, gen.ONES)
    for off in (0, 3):
        g, launches = _run(tcr, bits, off)
        assert launches == _levels(n), (n, launches)
        if n <= 32768:
            assert g == float(np.float16(n)), (n, off, g)


def test_empty_is_zero(tcr):
    g, launches = _run(tcr, np.zeros(0, dtype=np.uint16))
    assert g == 0.0 and launches == 0


def test_fp16_overflow_is_the_papers_open_precision_question(tcr):
    """65536 ones: the last level adds 256 partials of 256 in binary16 and
    the total 65536 exceeds binary16's 65504 -> inf (P:273 'precision loss')."""
    g, _ = _run(tcr, gen.generate(0, 0, 65536, gen.ONES))
    assert g == math.inf


def test_small_integers_exact_while_representable(tcr):
    # {-1, 0, 1} data with 4096 elements: every partial is an integer of
    # magnitude <= 256 (group) and the total <= 4096 is exact if each level
    # sum stays <= 2048 in magnitude -- checked against the oracle directly
    rng = np.random.default_rng(3)
    for case in range(20):
        v = rng.integers(-1, 2, 4096).astype(np.float16)
        bits = v.view(np.uint16)
        es = oracle.exact_sum_fp16(bits)
        g, _ = _run(tcr, bits)
        assert g == es.f32(), (case, g, es.f64())


def test_uniform_error_is_bounded_by_fp16_roundings(tcr):
    """uniform[-1,1]: the literal algorithm is accurate to a few binary16
    roundings per level, not to the fp32 budget (recorded by the precision study)."""
    for n in (4096, 1 << 16, 1 << 20):
        bits = gen.generate(gen.SEED_C1, 0, n, gen.UNIFORM_PM1)
        es = oracle.exact_sum_fp16(bits)
        g, _ = _run(tcr, bits)
        # per level: <= 2 roundings of 2^-11 relative on partials bounded by sum|x|
        bound = 2 * _levels(n) * 2.0 ** -11 * float(es.abs_value) * 2
        assert abs(g - es.f64()) <= bound, (n, g, es.f64(), bound)
