"""Host-side decoders of the exact kernels' integer state (test helpers only).

The product path never needs these: tcr_exact_finalize_ex rounds the state
on the device.  The tests use them to compare the raw state with the
oracle's exact T bit for bit.  Layouts are those include/tcr.h documents.
"""
from fractions import Fraction


def exact_limbs_to_int(acc) -> int:
    """T (units of 2^-24 for binary16; the type's unit for fp8) from the
    limbs l0, l1, l2 of an acc[6] state: T = l0 + l1 * 2^40 + l2 * 2^80."""
    a = [int(v) for v in (acc.tolist() if hasattr(acc, "tolist") else acc)]
    return a[0] + (a[1] << 40) + (a[2] << 80)


def exact_bf16_windows_to_value(acc) -> Fraction:
    """Exact rational value of a bfloat16 exact state (27 int64): window k
    holds I_k = a[3k] + a[3k+1] * 2^40 + a[3k+2] * 2^80 in units of 2^-133
    (k = 0) or 2^(32k - 134) (k >= 1)."""
    a = [int(v) for v in (acc.tolist() if hasattr(acc, "tolist") else acc)]
    tot = Fraction(0)
    for k in range(8):
        i_k = a[3 * k] + (a[3 * k + 1] << 40) + (a[3 * k + 2] << 80)
        unit = Fraction(1, 1 << 133) if k == 0 else Fraction(2) ** (32 * k - 134)
        tot += i_k * unit
    return tot
