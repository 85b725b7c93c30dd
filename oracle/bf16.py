"""bfloat16 rounding for the oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

The layer stores activations in bf16 (BASELINE north_star: "bf16 storage, fp32
accumulate"; reading G5 in DESIGN.md: h and Y are each rounded once, RNE).  The
oracle keeps every value in float64 and rounds at exactly those storage points
with the function below.

bf16 = 1 sign bit, 8 exponent bits (same range as IEEE binary32), 7 stored
significand bits.  Rounding is IEEE round-to-nearest, ties-to-even, applied
directly to the float64 value (no intermediate float32 rounding, so there is no
double rounding).
"""

import numpy as np

_BF16_MAX = float.fromhex("0x1.fep127")     # largest finite bf16
_MIN_NORMAL = 2.0 ** -126                    # smallest normal bf16 (= fp32)
_SUBNORMAL_QUANTUM = 2.0 ** -133             # bf16 subnormal spacing


def round_to_bf16(x):
    """Round float64 values to the nearest bf16 value (ties to even).

    Returns float64 values that are exactly representable in bf16.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    a = np.abs(x)

    normal = np.isfinite(x) & (a >= _MIN_NORMAL)
    # Normal range: keep 8 significant bits of the 53-bit float64 significand.
    # Drop the low 45 fraction bits with round-half-to-even on the integer bits.
    bits = x[normal].view(np.uint64)
    drop = np.uint64(45)
    lsb = (bits >> drop) & np.uint64(1)
    bits = bits + (np.uint64((1 << 44) - 1) + lsb)
    bits = bits & ~np.uint64((1 << 45) - 1)
    r = bits.view(np.float64)
    r = np.where(np.abs(r) > _BF16_MAX, np.copysign(np.inf, r), r)
    out[normal] = r

    sub = np.isfinite(x) & (a < _MIN_NORMAL)
    # Subnormal range: fixed spacing 2^-133; np.round is half-to-even.
    out[sub] = np.round(x[sub] / _SUBNORMAL_QUANTUM) * _SUBNORMAL_QUANTUM

    nonfinite = ~np.isfinite(x)
    out[nonfinite] = x[nonfinite]
    return out


def to_bits(x):
    """bf16 bit patterns (uint16) of float64 values already rounded to bf16."""
    r = round_to_bf16(x)
    return (r.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bits(u16):
    """float64 values of bf16 bit patterns (uint16 array)."""
    u = np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)
