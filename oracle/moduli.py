"""Moduli families, P, q_l and the CRT weights.

* INT8 family: "scanning downward from 256 and greedily selecting
  integers that remain pairwise coprime to all previously selected values".
* Karatsuba family: the same greedy rule "in descending order starting
  from 513".
* Hybrid family (eq. p_list_hybrid): "we first prioritize square moduli
  by selecting pairwise coprime squares in descending order from 1089.  We then
  continue the list with pairwise coprime integers in descending order without
  restricting them to be squares."  Squares are limited to s^2 with s <= 33 (the
  digit rule needs |digits| <= 16) and non-squares to p <= 513
  (eq. limit1).  Reading R1: the square scan runs over
  s = 33, 32, ..., 2 keeping s^2 iff coprime to the kept squares, but only squares
  larger than 513 are taken (exactly the six printed ones; smaller squares would be
  dominated by the greedy tail); the non-square scan starts at 513.
  This reproduces the printed prefix P:309-313 and puts the seventh square
  (361 = 19^2) at index 33, which is why the paper assumes N < 34.
* P = prod p_l; q_l with q_l P/p_l = 1 (mod p_l); the CRT weight
  w_l = q_l P/p_l of eq. (CRT_finalreduction).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math
from dataclasses import dataclass
from fractions import Fraction

from . import fp32


def _greedy(start: int, count: int, kept=None, lowest: int = 2):
    kept = list(kept or [])
    c = start
    out = []
    while len(out) < count and c >= lowest:
        if all(math.gcd(c, q) == 1 for q in kept):
            kept.append(c)
            out.append(c)
        c -= 1
    if len(out) < count:
        raise ValueError("greedy scan exhausted")
    return out


def int8_moduli(N: int):
    """First N INT8-family moduli (eq. p_list)."""
    return _greedy(256, N)


def karatsuba_moduli(N: int):
    """First N Karatsuba-family moduli (eq. p_list_karatsuba)."""
    return _greedy(513, N)


def hybrid_squares():
    """Pairwise coprime squares s^2 > 513 with s <= 33, descending."""
    out = []
    for s in range(33, 1, -1):
        p = s * s
        if p <= 513:
            break
        if all(math.gcd(p, q) == 1 for q in out):
            out.append(p)
    return out


def hybrid_moduli(N: int):
    """First N hybrid moduli (eq. p_list_hybrid)."""
    if not 2 <= N <= 33:
        raise ValueError("hybrid moduli: N must be in [2, 33] (P:526 assumes N < 34)")
    sq = hybrid_squares()
    if N <= len(sq):
        return sq[:N]
    return sq + _greedy(513, N - len(sq), kept=sq)


def is_square(p: int) -> bool:
    s = math.isqrt(p)
    return s * s == p


@dataclass(frozen=True)
class CrtPlan:
    moduli: tuple
    P: int
    q: tuple        # q_l in [1, p_l)
    w: tuple        # w_l = q_l * P / p_l


def crt_plan(moduli) -> CrtPlan:
    """P, q_l and w_l of eq. (CRT_finalreduction)."""
    P = 1
    for p in moduli:
        P *= p
    qs, ws = [], []
    for p in moduli:
        Pp = P // p
        q = pow(Pp % p, -1, p)          # q_l P/p_l = 1 (mod p_l)
        qs.append(q)
        ws.append(q * Pp)
    return CrtPlan(tuple(moduli), P, tuple(qs), tuple(ws))


def smod(x: int, p: int) -> int:
    """Symmetric modulo.  Reading R2: range [-floor(p/2), ceil(p/2) - 1],
    i.e. [-(p-1)/2, (p-1)/2] for odd p and [-p/2, p/2 - 1] for even p."""
    r = x % p
    if 2 * r >= p:
        r -= p
    return r


def log2_big(x: int, frac_bits: int = 80) -> Fraction:
    """log2 of a positive integer to within 2^-frac_bits (floor), exactly enough to
    decide binary32 rounding of (log2(P-1) - 1)/2 with a checked margin."""
    # log2 x = e + log2(x / 2^e); compute log2 of the mantissa by the
    # square-and-compare bit-by-bit method on exact rationals.
    e = x.bit_length() - 1
    m = Fraction(x, 2 ** e)        # in [1, 2)
    bits = 0
    for _ in range(frac_bits):
        m = m * m
        bits <<= 1
        if m >= 2:
            m /= 2
            bits |= 1
        # keep the rational small: truncate to 200 bits (error far below 2^-frac_bits)
        if m.denominator.bit_length() > 400:
            m = Fraction(math.floor(m * 2 ** 300), 2 ** 300)
    return Fraction(e) + Fraction(bits, 2 ** frac_bits)


def p_prime(P: int) -> Fraction:
    """P' = FP32 round-down of (log2(P-1) - 1)/2."""
    lo = (log2_big(P - 1) - 1) / 2          # within 2^-80 below the true value
    hi = lo + Fraction(1, 2 ** 79)
    r = fp32.round_down(lo)
    if fp32.round_down(hi) != r:
        raise ArithmeticError("P' rounding undecided at 2^-80 precision")
    return r


def delta() -> Fraction:
    """delta = FP32 round-down of -1/(2 - 2^-21)."""
    return fp32.round_down(Fraction(-1) / (2 - Fraction(1, 2 ** 21)))


def effective_bits(moduli) -> float:
    """log2 sqrt(P/2) (Table 2)."""
    P = 1
    for p in moduli:
        P *= p
    return float(log2_big(P) - 1) / 2
