"""Correctly directed rounding of exact rationals to IEEE binary32.

Sec. III-E computes C-bar "in round-up mode" and evaluates
P' + delta*log2(max c-bar) "using FP32 arithmetic in round-down mode",
with P' and delta the "FP32 round-down values" of their real definitions
(P:379-380).  This module writes those roundings out: a binary32 value is
sign * M * 2^E with integer 2^23 <= M < 2^24 (normal) or the subnormal grid
2^-149 * M; we locate the neighbours of q exactly and pick the directed one.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math
import struct
from fractions import Fraction

_MIN_SUB = Fraction(1, 2 ** 149)
_MAX_F32 = Fraction((2 ** 24 - 1) * 2 ** 104)


def f32_bits(x: Fraction) -> int:
    """Bit pattern of a Fraction that is exactly a binary32 value."""
    f = float(x)
    assert Fraction(f) == x, "not exactly representable in binary64"
    b = struct.unpack("<I", struct.pack("<f", f))[0]
    assert Fraction(struct.unpack("<f", struct.pack("<I", b))[0]) == x, "not a binary32 value"
    return b


def from_bits(b: int) -> Fraction:
    return Fraction(struct.unpack("<f", struct.pack("<I", b & 0xFFFFFFFF))[0])


def _grid_exponent(a: Fraction) -> int:
    """Exponent E of the binary32 grid spacing 2^E around a > 0 (ulp = 2^E)."""
    # floor(log2 a) exactly
    n, d = a.numerator, a.denominator
    e = n.bit_length() - d.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    # normal numbers have 24-bit significands; subnormal grid is 2^-149
    return max(e - 23, -149)


def round_down(q) -> Fraction:
    """Largest binary32 value <= q (round toward -inf)."""
    q = Fraction(q)
    if q == 0:
        return Fraction(0)
    if q < 0:
        return -round_up(-q)
    if q > _MAX_F32:
        return _MAX_F32
    ulp = Fraction(2) ** _grid_exponent(q)
    return math.floor(q / ulp) * ulp


def round_up(q) -> Fraction:
    """Smallest binary32 value >= q (round toward +inf); overflow raises."""
    q = Fraction(q)
    if q == 0:
        return Fraction(0)
    if q < 0:
        return -round_down(-q)
    if q > _MAX_F32:
        raise OverflowError("round_up beyond FLT_MAX")
    ulp = Fraction(2) ** _grid_exponent(q)
    r = math.ceil(q / ulp) * ulp
    return r


def round_nearest(q) -> Fraction:
    """Round to nearest, ties to even (used by the oracle's model of an FP32 MMA)."""
    q = Fraction(q)
    if q == 0:
        return Fraction(0)
    if q < 0:
        return -round_nearest(-q)
    lo = round_down(q)
    if lo == q:
        return q
    hi = round_up(q)
    if q - lo < hi - q:
        return lo
    if q - lo > hi - q:
        return hi
    ulp = Fraction(2) ** _grid_exponent(lo)
    return lo if (lo / ulp) % 2 == 0 else hi
