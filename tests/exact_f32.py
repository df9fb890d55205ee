"""Exact-rational IEEE-754 binary32 rounding, used to pin the oracle.

Independent of both the oracle (no float32 multiply anywhere) and the CUDA
path: values are carried as ``fractions.Fraction`` and rounded once to the
nearest binary32, ties to even, with gradual underflow (subnormals) and
overflow to infinity -- the definition of a correctly rounded operation
(IEEE-754-2008 section 4.3.1 / 7.4).
"""
from __future__ import annotations

import struct
from fractions import Fraction

import numpy as np

EMIN = -126
PREC = 24                     # significand bits incl. hidden bit
MAX_EXP = 127
OVERFLOW = Fraction(2) ** (MAX_EXP + 1)


def f32_to_fraction(x) -> Fraction:
    x = np.float32(x)
    if not np.isfinite(x):
        raise ValueError("non-finite")
    return Fraction(float(x))          # float32 -> float64 is exact


def bits_to_f32(b: int) -> np.float32:
    return np.frombuffer(struct.pack("<I", b & 0xFFFFFFFF), dtype=np.float32)[0]


def f32_bits(x) -> int:
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


def _floor_log2(a: Fraction) -> int:
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    if Fraction(2) ** (e + 1) <= a:
        e += 1
    return e


def round_f32(v: Fraction, sign_of_zero: int = 1) -> np.float32:
    """Round an exact rational to binary32, RNE.  ``sign_of_zero`` gives the
    sign of an exact zero result (IEEE: product sign = xor of operand signs)."""
    if v == 0:
        return np.float32(0.0) if sign_of_zero > 0 else np.float32(-0.0)
    s = -1 if v < 0 else 1
    a = -v if v < 0 else v
    e = max(_floor_log2(a), EMIN)
    q = Fraction(2) ** (e - (PREC - 1))          # quantum (ulp) at this binade
    n = a / q
    fl = n.numerator // n.denominator
    rem = n - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    r = fl * q
    if r >= OVERFLOW:
        return np.float32(np.inf * s)
    if r == 0:                                    # underflow to zero keeps the sign
        return np.float32(0.0) if s > 0 else np.float32(-0.0)
    return np.float32(float(r) * s)


def mul(x, f) -> np.float32:
    """Correctly rounded binary32 product."""
    x, f = np.float32(x), np.float32(f)
    sign = -1 if (np.signbit(x) != np.signbit(f)) else 1
    return round_f32(f32_to_fraction(x) * f32_to_fraction(f), sign)


def axpy(a, x, y) -> np.float32:
    """fl(fl(a*x) + y): the two-rounding AXPY (no fused multiply-add)."""
    p = mul(a, x)
    s = f32_to_fraction(p) + f32_to_fraction(y)
    # IEEE: exact zero sum of opposite-signed operands is +0 in RNE
    sign = 1 if s != 0 or not (np.signbit(p) and np.signbit(np.float32(y))) else -1
    return round_f32(s, sign)


def fma(a, x, y) -> np.float32:
    """fl(a*x + y) with a single rounding (what contraction would compute)."""
    s = f32_to_fraction(a) * f32_to_fraction(x) + f32_to_fraction(y)
    return round_f32(s, 1)
