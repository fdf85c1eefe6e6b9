"""Pins for oracle.model: the paper's R_tc structure and cost model (CPU only).

Pinned by the values PAPER.md prints (tests/golden/paper_model.json), SPEC.md
worked examples (tests/golden/spec_examples.json), closed forms and
invariants.  The exact C oracle (a different algorithm) must agree with R_tc.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tcr_inputs as gen
from oracle import model as M


def _seq(spec):
    if spec == "1..16":
        return list(range(1, 17))
    return spec


def _mat(v, m):
    if v == "ones":
        return M.ones(m)
    if v == "zeros":
        return M.zeros(m)
    return np.array(v, dtype=object)


# ---------------- paper-printed values ----------------

def test_paper_speedups(paper_golden):
    for ex in paper_golden["speedup_values"]:
        assert M.speedup(ex["m"]) == Fraction(ex["S"])
        assert float(M.speedup(ex["m"])) == float(ex["printed"])
    assert M.speedup(2) > 1


def test_paper_base_case_five_units(paper_golden):
    for m in paper_golden["tc_base_case"]["m"]:
        led = M.CostLedger()
        x = list(range(1, m * m + 1))
        assert M.reduce_tensor(x, m, led) == sum(x)
        assert led.total_time == 5
        assert led.trace == ["coalesced_read", "tile_rw", "mma_cycle", "mma_cycle", "tile_rw"]
        assert M.predict_tensor(m * m, m) == 5


def test_closed_form_matches_ledger_powers():
    # ledger == 5*log_{m^2} n for n = (m^2)^k; classic 4*log2 n.
    for m, kmax in ((2, 5), (4, 3), (16, 2)):
        for k in range(1, kmax + 1):
            n = (m * m) ** k
            led = M.CostLedger()
            x = [1] * n
            assert M.reduce_tensor(x, m, led) == n
            assert led.total_time == 5 * k == M.predict_tensor(n, m)
            assert abs(M.tc_steps_real(n, m) - 5 * k) < 1e-9
            assert led.noncoalesced_rw == 0
    for j in range(1, 13):
        led = M.CostLedger()
        assert M.reduce_pairwise([1] * (1 << j), led) == 1 << j
        assert led.total_time == 4 * j == M.predict_classic(1 << j)


def test_speedup_ratio_exact_at_65536(spec_golden):
    ex = spec_golden["acceptance_n65536"]
    lt, lc = M.CostLedger(), M.CostLedger()
    x = [1] * ex["n"]
    M.reduce_tensor(x, ex["m"], lt)
    M.reduce_pairwise(x, lc)
    assert lt.total_time == ex["tensor_units"] and lc.total_time == ex["classic_units"]
    assert Fraction(lc.total_time, lt.total_time) == Fraction(ex["ratio"]) == M.speedup(16)


# ---------------- SPEC worked examples ----------------

def test_spec_mma_examples(spec_golden):
    for ex in spec_golden["mma"]:
        m = ex["m"]
        D = M.mma(_mat(ex["A"], m), _mat(ex["B"], m), _mat(ex["C"], m))
        assert D.tolist() == ex["D"]
    A = np.array([[1, 2], [3, 4]], dtype=object)
    assert M.mma(M.zeros(2), A, A).tolist() == A.tolist()  # zero annihilates
    with pytest.raises(ValueError):
        M.mma(M.ones(2), M.ones(3), M.zeros(2))


def test_spec_load_group(spec_golden):
    for ex in spec_golden["load_group"]:
        assert M.load_group(_seq(ex["X"]), ex["offset"], ex["m"]).tolist() == ex["A"]


def test_spec_mma_reduce_group(spec_golden):
    for ex in spec_golden["mma_reduce_group"]:
        led = M.CostLedger()
        assert M.mma_reduce_group(np.array(ex["A"], dtype=object), led, check=True) == ex["result"]
        assert led.mma_cycles == 2 and led.mma_ops == 2


def test_spec_reduce_tensor(spec_golden):
    for ex in spec_golden["reduce_tensor"]:
        x = _seq(ex["X"])
        m = ex["m"]
        assert M.reduce_tensor(x, m) == ex["result"]
        if "level1" in ex:
            lv1 = [M.mma_reduce_group(M.load_group(x, g * m * m, m)) for g in range(len(ex["level1"]))]
            assert lv1 == ex["level1"]


def test_spec_partition(spec_golden):
    for ex in spec_golden["partition"]:
        p = M.partition(ex["n"], ex["m"])
        assert p.total_levels == ex["levels"]
        if "groups" in ex:
            assert [lv.groups for lv in p.levels] == ex["groups"]
        if "padded" in ex:
            assert [lv.padded_slots for lv in p.levels] == ex["padded"]
    with pytest.raises(ValueError):
        M.partition(10, 1)


def test_spec_pairwise(spec_golden):
    for ex in spec_golden["reduce_pairwise"]:
        led = M.CostLedger()
        assert M.reduce_pairwise(_seq(ex["X"]), led) == ex["result"]
        assert led.total_time == ex["units"]


def test_spec_predictors(spec_golden):
    for ex in spec_golden["predict_classic"]:
        assert M.predict_classic(ex["n"]) == ex["steps"]
    for ex in spec_golden["predict_tensor"]:
        assert M.predict_tensor(ex["n"], ex["m"]) == ex["steps"]
    for ex in spec_golden["speedup"]:
        assert M.speedup(ex["m"]) == Fraction(ex["S"])
    for ex in spec_golden["parallel_cost"]:
        assert M.parallel_cost(ex["steps"], ex["p"]) == ex["cost"]
    for ex in spec_golden["brent_bound"]:
        assert M.brent_bound(ex["n"], ex["p"]) == ex["bound"]
    with pytest.raises(ValueError):
        M.predict_tensor(1, 16)


def test_brent_efficient_cost():
    # Eq. 6-7: p = n/log2 n gives C_p = O(n), here <= 2n.
    for k in range(4, 21):
        n = 1 << k
        p = n / k
        assert M.parallel_cost(M.brent_bound(n, p), p) <= 2 * n


# ---------------- invariants ----------------

@pytest.mark.parametrize("m", [2, 4, 8, 16])
def test_replication_invariants_random_tiles(m):
    # Eq. 10 column replication and Eq. 12 full replication, exact.
    rng = np.random.default_rng(m)
    for _ in range(50):
        vals = gen.generate(int(rng.integers(1 << 30)), 0, m * m, gen.WIDE)
        A = M.load_group(vals.view(np.float16).astype(np.float64).tolist(), 0, m)
        M.mma_reduce_group(A, check=True)


def test_oracle_equivalence_random():
    # reduce_tensor == reduce_pairwise == reduce_sequential == exact C oracle.
    rng = np.random.default_rng(42)
    for case in range(40):
        n = int(rng.integers(0, 3000))
        m = int(rng.integers(2, 17))
        x = gen.generate(case, 0, n, gen.WIDE)
        vals = x.view(np.float16).astype(np.float64).tolist()
        exact = oracle.exact_sum_fp16(x).value
        assert M.reduce_tensor(vals, m) == exact
        assert M.reduce_pairwise(vals) == exact
        assert M.reduce_sequential(vals) == exact


def test_padding_permutation_and_mma_count():
    rng = np.random.default_rng(7)
    for case in range(20):
        n = int(rng.integers(1, 2000))
        m = int(rng.integers(2, 9))
        vals = gen.generate(case, 0, n, gen.UNIFORM_PM1).view(np.float16).astype(np.float64).tolist()
        led = M.CostLedger()
        r = M.reduce_tensor(vals, m, led)
        assert M.reduce_tensor(vals + [0.0] * int(rng.integers(1, 50)), m) == r
        assert M.reduce_tensor(list(rng.permutation(vals)), m) == r
        plan = M.partition(n, m)
        assert led.levels == plan.total_levels
        assert led.mma_ops == 2 * sum(lv.groups for lv in plan.levels)
