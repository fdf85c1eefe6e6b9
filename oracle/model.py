"""oracle.model -- TEST INFRASTRUCTURE ONLY.

The paper's algorithm and cost model, step by step in the paper's order and
notation, in exact arithmetic (Python ints / ``fractions.Fraction``; numpy
``object`` arrays so that ``@`` is exact).  Used to pin the *structure* of
the method (groups, levels, padding, the two-MMA algebra, step counts), which
the GPU path realises with a different, fused hierarchy.

Citations are PAPER.md line numbers ("P:L") and SPEC.md line numbers ("S:L").

* :func:`mma` -- D = A x B + C (Eq. 8), charged 1 cycle.
* :func:`load_group` -- m^2 consecutive elements into A row-major, "A_{m,m} is
  the m^2-th element of the group", zero padding.
* :func:`mma_reduce_group` -- D = A x 1 + 0 (Eq. 9-10), then
  D' = 1 x D + 0 (Eq. 11-12), read D'_{1,1}.
* :func:`reduce_tensor` -- R_tc (Eq. 13-14), level by level.
* :func:`reduce_pairwise` -- classic x_i + x_{i+n/2^k} tree.
* :func:`partition`, :func:`predict_tensor`, :func:`predict_classic`,
  :func:`speedup`, :func:`tc_steps_real`, :func:`parallel_cost`,
  :func:`brent_bound` -- Eq. 4-7 and 15-17.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

# --------------------------------------------------------------------------
# Cost model: coalesced r/w = 1, non-coalesced r/w = w,
# tensor-core MMA = 1 cycle, simultaneous r/w into tensor-core matrices = 1.
# --------------------------------------------------------------------------


@dataclass
class CostLedger:
    """Counts of simulated time units per operation class.

    Charges are *parallel* time: one charge per level for an operation that
    all groups of the level perform simultaneously ("simultaneously
    for all the m^2 groups").  ``mma_ops`` separately counts every MMA
    executed (2 per group).
    """

    coalesced_rw: int = 0
    noncoalesced_rw: int = 0
    tile_rw: int = 0
    mma_cycles: int = 0
    classic_add: int = 0
    classic_store: int = 0
    w: int = 32  # never charged by either algorithm; reading G16
    mma_ops: int = 0
    levels: int = 0
    trace: list = field(default_factory=list)

    def charge(self, op: str) -> None:
        if op == "coalesced_read" or op == "coalesced_write":
            self.coalesced_rw += 1
        elif op == "noncoalesced_read":
            self.noncoalesced_rw += 1
        elif op == "tile_rw":
            self.tile_rw += 1
        elif op == "mma_cycle":
            self.mma_cycles += 1
        elif op == "classic_add":
            self.classic_add += 1
        elif op == "classic_store":
            self.classic_store += 1
        else:
            raise ValueError(f"unknown op class {op!r}")
        self.trace.append(op)

    @property
    def total_time(self) -> int:
        return (self.coalesced_rw + self.noncoalesced_rw * self.w + self.tile_rw
                + self.mma_cycles + self.classic_add + self.classic_store)


# --------------------------------------------------------------------------
# Tiles and the MMA primitive (Eq. 8)
# --------------------------------------------------------------------------


def ones(m: int) -> np.ndarray:
    """The all-ones m x m matrix of Eq. 9 ("B_{m x m} as an all-ones matrix")."""
    return np.array([[1] * m for _ in range(m)], dtype=object)


def zeros(m: int) -> np.ndarray:
    """The zero m x m matrix of Eq. 9 ("C is a zero-matrix")."""
    return np.array([[0] * m for _ in range(m)], dtype=object)


def _exact(v):
    """Exact scalar: ints stay ints, floats become their exact Fraction."""
    if isinstance(v, (int, Fraction)):
        return v
    if isinstance(v, (np.integer,)):
        return int(v)
    return Fraction(float(v))


def mma(A: np.ndarray, B: np.ndarray, C: np.ndarray, ledger: CostLedger | None = None) -> np.ndarray:
    """D = A x B + C (Eq. 8), exact; one MMA cycle."""
    if A.shape != B.shape or A.shape != C.shape or A.shape[0] != A.shape[1]:
        raise ValueError("mma: A, B, C must all be m x m")
    D = A.dot(B) + C  # object dtype: exact Python arithmetic
    if ledger is not None:
        ledger.charge("mma_cycle")
        ledger.mma_ops += 1
    return D


def load_group(X, offset: int, m: int) -> np.ndarray:
    """A_{m x m} from X[offset .. offset+m^2), row-major, zero-padded."""
    if m < 2:
        raise ValueError("m must be >= 2 (P:262)")
    A = zeros(m)
    for k in range(m * m):
        if offset + k < len(X):
            A[k // m][k % m] = _exact(X[offset + k])
    return A


def mma_reduce_group(A: np.ndarray, ledger: CostLedger | None = None, check: bool = False):
    """Two-step MMA group reduction (Eq. 9-12); returns D'_{1,1}.

    With ``check=True`` asserts the replication invariants the paper states:
    every column of D holds the row sums (Eq. 10) and every entry of
    D' holds the group total (Eq. 12).
    """
    m = A.shape[0]
    one, zero = ones(m), zeros(m)
    D = mma(A, one, zero, ledger)          # Eq. 9-10: row sums in every column
    Dp = mma(one, D, zero, ledger)         # Eq. 11-12: "D in the position of B, ones in A"
    if check:
        for i in range(m):
            rs = sum(A[i][k] for k in range(m))
            assert all(D[i][j] == rs for j in range(m)), "Eq. 10 column replication"
        tot = sum(A[i][k] for i in range(m) for k in range(m))
        assert all(Dp[i][j] == tot for i in range(m) for j in range(m)), "Eq. 12 replication"
    return Dp[0][0]


# --------------------------------------------------------------------------
# Reduction plan and algorithms (Eq. 13-14)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Level:
    size: int          # problem size entering the level
    groups: int        # ceil(size / m^2)
    padded_slots: int  # groups * m^2 - size (zero padding)


@dataclass(frozen=True)
class ReductionPlan:
    n: int
    m: int
    levels: tuple

    @property
    def total_levels(self) -> int:
        return len(self.levels)


def partition(n: int, m: int) -> ReductionPlan:
    """Levels of R_tc: size_{k+1} = ceil(size_k / m^2) until one value.

    0 levels for n <= 1; 1 level for 2 <= n <= m^2 (Eq. 14).
    """
    if m < 2:
        raise ValueError("m must be >= 2 (P:262)")
    if n < 0:
        raise ValueError("n must be >= 0")
    g2 = m * m
    levels = []
    size = n
    while size > 1:
        groups = -(-size // g2)
        levels.append(Level(size, groups, groups * g2 - size))
        size = groups
    return ReductionPlan(n, m, tuple(levels))


def reduce_tensor(X, m: int, ledger: CostLedger | None = None, check: bool = False):
    """R_tc(X) (Eq. 13-14), exact.  Ledger: 5 units per level.

    Per level, in the paper's order: coalesced read (1), load into
    the tensor-core matrices (1), the two MMAs of every group (2, done
    "simultaneously for all the m^2 groups"), write D'_{1,1} of each group to
    its location in the next array (1).
    """
    ledger = ledger if ledger is not None else CostLedger()
    cur = [_exact(v) for v in X]
    if len(cur) == 0:
        return 0
    plan = partition(len(cur), m)
    for lv in plan.levels:
        ledger.charge("coalesced_read")
        ledger.charge("tile_rw")
        ledger.charge("mma_cycle")
        ledger.charge("mma_cycle")
        ledger.charge("tile_rw")  # the write of D'_{1,1} into X
        ledger.levels += 1
        nxt = []
        for gidx in range(lv.groups):
            A = load_group(cur, gidx * m * m, m)
            # the two MMAs are charged once per level above (parallel time);
            # count the executed MMAs separately
            nxt.append(mma_reduce_group(A, None, check))
            ledger.mma_ops += 2
        cur = nxt
    return cur[0]


def reduce_pairwise(X, ledger: CostLedger | None = None):
    """Classic tree: at step k thread i adds x_i + x_{i+n/2^k}.

    Non-powers of two are zero-padded to the next power (additive identity).
    Ledger: 4 units per level = read, read, add, store.
    """
    ledger = ledger if ledger is not None else CostLedger()
    cur = [_exact(v) for v in X]
    if len(cur) == 0:
        return 0
    size = 1
    while size < len(cur):
        size *= 2
    cur = cur + [0] * (size - len(cur))
    while size > 1:
        half = size // 2
        ledger.charge("coalesced_read")
        ledger.charge("coalesced_read")
        ledger.charge("classic_add")
        ledger.charge("classic_store")
        ledger.levels += 1
        cur = [cur[i] + cur[i + half] for i in range(half)]
        size = half
    return cur[0]


def reduce_sequential(X):
    """The Theta(n) single-accumulator loop, exact."""
    acc = 0
    for v in X:
        acc += _exact(v)
    return acc


# --------------------------------------------------------------------------
# Closed forms (Eq. 4-7, 15-17)
# --------------------------------------------------------------------------


def _ceil_log(n: int, base: int) -> int:
    """ceil(log_base(n)) for n >= 1, in integer arithmetic."""
    k, p = 0, 1
    while p < n:
        p *= base
        k += 1
    return k


def predict_tensor(n: int, m: int) -> int:
    """T_tc(n) = 5 * ceil(log_{m^2} n) (Eq. 16; ceiling per S:271)."""
    if n < 2 or m < 2:
        raise ValueError("domain: n >= 2, m >= 2")
    return 5 * _ceil_log(n, m * m)


def tc_steps_real(n: int, m: int) -> float:
    """T_tc(n) = 5 * log_{m^2}(n) without ceiling."""
    return 5.0 * math.log(n) / math.log(m * m)


def predict_classic(n: int) -> int:
    """T(n) = 4 * ceil(log2 n)."""
    if n < 2:
        raise ValueError("domain: n >= 2")
    return 4 * _ceil_log(n, 2)


def speedup(m: int):
    """S = (4/5) * log2(m^2) (Eq. 17).  Exact Fraction when m is a power of 2."""
    if m < 2:
        raise ValueError("m must be >= 2")
    if m & (m - 1) == 0:
        return Fraction(4, 5) * (2 * (m.bit_length() - 1))
    return 0.8 * math.log2(m * m)


def parallel_cost(steps, p):
    """C_p = T_p(n) * p."""
    return steps * p


def brent_bound(n: int, p) -> float:
    """T_p(n) <= T_1(n)/p + T_inf(n) with T_1 = n, T_inf = log2 n (Eq. 5)."""
    if n < 2 or p < 1:
        raise ValueError("domain: n >= 2, p >= 1")
    return n / p + math.log2(n)


__all__ = [
    "CostLedger", "Level", "ReductionPlan", "ones", "zeros", "mma", "load_group",
    "mma_reduce_group", "partition", "reduce_tensor", "reduce_pairwise",
    "reduce_sequential", "predict_tensor", "tc_steps_real", "predict_classic",
    "speedup", "parallel_cost", "brent_bound",
]
