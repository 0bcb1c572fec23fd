"""Exact two-sided pins for the accurate-mode scaling constants of eq. mu-computation
(P:374-381): the FP32 log2 (reading R7), P' = RD32((log2(P-1) - 1)/2) and
the safety factor f_k (reading R5), plus the fast-mode rule R15 against the
FP64-norm rule it replaces.

Each check brackets the oracle's value from BOTH sides against something computed
independently of it: ``decimal`` natural logarithms at 60-80 significant digits
(correctly rounded, no shared code with ``math.log2`` or ``oracle.moduli.log2_big``),
exact rational arithmetic, and hand-derived bit patterns (``tests/golden/
derived_constants.json``, each with its derivation).  A round-to-nearest log2, a P'
a few ulps low or an f_k a few ulps off each fails here.
"""
import math
import struct
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

from conftest import load_golden
from oracle import fp32, moduli as mod, scheme, fp8
from synth import gen_host


def _f32(bits: int) -> Fraction:
    return Fraction(struct.unpack("<f", struct.pack("<I", bits))[0])


def _bits(x: Fraction) -> int:
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def _next_up32(x: Fraction) -> Fraction:
    """The binary32 successor of a positive or negative binary32 value x."""
    b = _bits(x)
    if x > 0:
        return _f32(b + 1)
    if x == 0:
        return _f32(1)
    return _f32(b - 1)


def _dec_log2_int_ratio(num: int, den: int, digits: int) -> Decimal:
    """log2(num/den) to `digits` significant digits via decimal's correctly rounded ln."""
    getcontext().prec = digits + 10
    return (Decimal(num).ln() - Decimal(den).ln()) / Decimal(2).ln()


def _dec(q: Fraction) -> Decimal:
    return Decimal(q.numerator) / Decimal(q.denominator)


# ------------------------------------------------------------------ FP32 log2 (R7)

def _log2_cases():
    rng = np.random.default_rng(2024)
    # binary32 arguments over the range c-bar takes (k 2^-18 .. k 2^16 for k <= 2^16)
    xs = [Fraction(float(np.float32(v))) for v in np.exp2(rng.uniform(-18.0, 32.0, 400))]
    xs += [Fraction(3), Fraction(5), Fraction(7), Fraction(10), Fraction(2 ** 14),
           Fraction(2 ** 14 + 1), Fraction(2 ** 24 - 1), Fraction(float(np.float32(1 / 3072)))]
    return xs


def test_log2_rd32_is_round_down_of_exact_log2():
    """log2_rd32(c) = L must satisfy L <= log2 c < succ32(L) (decimal ln at 60 digits).

    About half of the random arguments have log2 c in the upper half of its binary32
    ulp, where round-to-nearest and round-down differ: asserted, so the sample really
    separates the two rules."""
    upper_half = 0
    for c in _log2_cases():
        L = scheme.log2_rd32(c)
        lg = _dec_log2_int_ratio(c.numerator, c.denominator, 60)
        lo, hi = _dec(L), _dec(_next_up32(L))
        if c.denominator == 1 and c.numerator & (c.numerator - 1) == 0:
            assert L == c.numerator.bit_length() - 1          # exact powers of two
            continue
        # R7 rounds binary64 log2 to binary32: the bracket holds unless log2 c lies
        # within one binary64 ulp of a binary32 boundary (never in this sample)
        margin = Decimal(2) ** -50 * max(abs(lg), Decimal(1))
        assert lo <= lg < hi, (c, L)
        assert lg - lo > margin and hi - lg > margin
        if (lg - lo) > (hi - lg):
            upper_half += 1
    assert upper_half > 100


def test_log2_rd32_hand_values():
    """Hand-derived bit patterns (derivation in the golden file): c = 7, 11, 17 discard
    0.88-0.98 ulp, so rounding to nearest would give the next pattern up; c = 3 discards
    0.11 ulp; 16384 is exact."""
    d = load_golden("derived_constants.json")["log2_rd32"]
    for case in d["cases"]:
        L = scheme.log2_rd32(Fraction(case["c"]))
        assert _bits(L) == int(case["bits_hex"], 16), case


# ------------------------------------------------------------------ P'

@pytest.mark.parametrize("family", ["hybrid", "karatsuba"])
def test_pprime_two_sided_all_N(family):
    """P' = RD32((log2(P-1) - 1)/2) for N = 2..33: P' <= v < succ32(P') with v from
    decimal ln at 80 digits (independent of log2_big's square-and-compare), and v not
    within 2^-60 of either end (so the bracket decides)."""
    for N in range(2, 34):
        P = math.prod(scheme.family_moduli(N, family))
        Pp = mod.p_prime(P)
        v = (_dec_log2_int_ratio(P - 1, 1, 80) - 1) / 2
        lo, hi = _dec(Pp), _dec(_next_up32(Pp))
        assert lo <= v < hi, (family, N)
        assert v - lo > Decimal(2) ** -60 and hi - v > Decimal(2) ** -60


def test_pprime_hand_value_N12_N13():
    """Bit patterns of P' for the headline N (derivation in the golden file)."""
    d = load_golden("derived_constants.json")["p_prime"]
    for case in d["cases"]:
        P = math.prod(mod.hybrid_moduli(case["N"]))
        assert _bits(mod.p_prime(P)) == int(case["bits_hex"], 16), case


# ------------------------------------------------------------------ f_k (R5)

def test_safety_factor_hand_bit_patterns():
    """f_k = RU32(1/(1 - k 2^-23)) at k = 4096, 16384, 65536 against hand-derived bits:
    1/(1 - 2^-j) = 1 + 2^-j + 2^-2j + 2^-3j + ..., truncated to 23 fraction bits and
    rounded up (the tail is nonzero)."""
    d = load_golden("derived_constants.json")["f_k"]
    for case in d["cases"]:
        assert _bits(scheme.safety_factor(case["k"])) == int(case["bits_hex"], 16), case


def test_safety_factor_two_sided():
    """f_k is the SMALLEST binary32 value >= 1/(1 - k 2^-23): the predecessor is below."""
    for k in [1, 2, 3, 100, 1000, 4095, 4096, 4097, 8192, 12345, 16384, 32768, 65535,
              65536, 2 ** 20, 2 ** 22]:
        f = scheme.safety_factor(k)
        exact_inv = Fraction(1) / (1 - Fraction(k, 2 ** 23))
        pred = _f32(_bits(f) - 1)
        assert pred < exact_inv <= f, k


# ------------------------------------------------------------------ full offset on a worked case

def test_offset_from_cbar_two_sided():
    """t = floor(RD32(P' + RD32(delta RD32(log2 cbar)))): each FP32 step recomputed
    independently (decimal log2, exact rational products/sums rounded down by hand via
    the binary32 grid) for random cbar at N = 12, 13."""
    rng = np.random.default_rng(5)
    dlt = mod.delta()
    for N in (12, 13):
        Pp = mod.p_prime(math.prod(mod.hybrid_moduli(N)))
        for v in np.exp2(rng.uniform(0.0, 40.0, 60)):
            cbar = Fraction(float(np.float32(v)))
            # independent round-down onto the binary32 grid
            def rd(q):
                q = Fraction(q)
                x = Fraction(float(np.float32(float(q))))
                while x > q:
                    x = _f32(_bits(x) - 1) if x > 0 else -_f32(_bits(-x) + 1)
                while _next_up32(x) <= q:
                    x = _next_up32(x)
                return x
            lg = _dec_log2_int_ratio(cbar.numerator, cbar.denominator, 60)
            x1 = Fraction(float(np.float32(float(lg))))
            while _dec(x1) > lg:
                x1 = _f32(_bits(x1) - 1) if x1 > 0 else -_f32(_bits(-x1) + 1)
            while _dec(_next_up32(x1)) <= lg:
                x1 = _next_up32(x1)
            x2 = rd(dlt * x1)
            x3 = rd(Pp + x2)
            assert scheme.offset_from_cbar(cbar, Pp, dlt) == math.floor(x3)


# ------------------------------------------------------------------ fast mode R15 vs S:286

def _spec_norm_exponent(row, P):
    """SPEC's FP64-norm rule evaluated exactly: the largest e with
    2^e n_i <= sqrt((P-1)/2), n_i = ||a_i||_2 (1 + 2^-30), i.e. 2^(2e) n_i^2 <= (P-1)/2."""
    n2 = sum((Fraction(float(v)) ** 2 for v in row), Fraction(0)) * (1 + Fraction(1, 2 ** 30)) ** 2
    X = Fraction(P - 1, 2)
    e = math.floor((math.log2(X) - math.log2(n2)) / 2) + 1
    while Fraction(2) ** (2 * e) * n2 > X if e >= 0 else n2 > X * Fraction(2) ** (-2 * e):
        e -= 1
    while (Fraction(2) ** (2 * (e + 1)) * n2 <= X) if e + 1 >= 0 else (n2 <= X * Fraction(2) ** (-2 * (e + 1))):
        e += 1
    return e


@pytest.mark.parametrize("phi,k", [(0.0, 64), (1.0, 300), (4.0, 200), (2.0, 2048)])
def test_fast_exponents_within_one_of_norm_rule(phi, k):
    """Reading R15 bounds with the FP8 upper bounds a-bar >= |mu' a| instead of |a|: its
    exponents never exceed the FP64-norm rule's and are at most 1 below it (a-bar <= 9/8
    |mu' a| above the E4M3 subnormal range, so the sum of squares grows by < 4x).  This
    is DESIGN.md's "<= 0.17 bit" claim, checked exactly."""
    N = 13
    plan, _, _ = scheme.plan_constants(N)
    A = gen_host(24, k, "phi", phi=phi, seed=91, order="C")
    e_prime, codes = scheme.prescale_rows(A)
    e_fast = scheme.fast_exponents(e_prime, codes, plan, [False] * A.shape[0])
    below = 0
    for i in range(A.shape[0]):
        e_norm = _spec_norm_exponent(A[i], plan.P)
        assert e_norm - 1 <= e_fast[i] <= e_norm, (i, e_fast[i], e_norm)
        below += e_fast[i] < e_norm
    assert below < A.shape[0]          # mostly equal: the loss is a fraction of a bit


# ------------------------------------------------------------------ more hand pins (mutation sweep)

def test_cbar_is_round_up_of_fk_R():
    """c-bar = RU32(f_k R) ("in round-up mode"): c-bar >= f_k R and its binary32
    predecessor is below, for R on and off the binary32 grid (R itself is an FP32 value)."""
    rng = np.random.default_rng(11)
    for k in (1000, 16384, 65536):
        fk = scheme.safety_factor(k)
        for v in np.exp2(rng.uniform(0.0, 34.0, 50)):
            R = Fraction(float(np.float32(v)))
            c = scheme.cbar_of(R, k)
            assert c >= fk * R and _f32(_bits(c) - 1) < fk * R


def test_square_digit_ties_are_round_half_even():
    """Reading R9 ("round", ties to even).  Ties occur only for p = 1024 (s = 32) at
    r = 16 (mod 32): r = 16 -> 16/32 = 0.5 -> D1 = 0, D2 = 16; r = 48 -> 1.5 -> D1 = 2,
    D2 = -16; r = -16 -> -0.5 -> D1 = 0, D2 = -16; r = 80 -> 2.5 -> D1 = 2, D2 = 16;
    r = -48 -> -1.5 -> D1 = -2, D2 = 16 (worked by hand)."""
    want = {16: (0, 16), 48: (2, -16), -16: (0, -16), 80: (2, 16), -48: (-2, 16), 17: (1, -15)}
    for r, d in want.items():
        assert scheme.digits_square(r, 32) == d, r


def test_mma_model_is_round_to_nearest_even():
    """Reading R6: the bound GEMM's FP32 result is modelled as the exact sum rounded once to
    nearest-even binary32.  In units of 2^-18, binary32 spacing is 4 in [2^25, 2^26) and 8
    in [2^26, 2^27): 2^25 + 3 -> 2^25 + 4 (nearer; round-down would give 2^25); the ties
    2^25 + 2 -> 2^25 (significand 2^23, even) and 2^25 + 6 -> 2^25 + 8 (2^23 + 2, even);
    2^26 + 5 -> 2^26 + 8; 2^26 + 3 -> 2^26 (worked by hand)."""
    u = Fraction(1, 2 ** 18)
    want = {2 ** 25 + 3: 2 ** 25 + 4, 2 ** 25 + 2: 2 ** 25, 2 ** 25 + 6: 2 ** 25 + 8,
            2 ** 26 + 5: 2 ** 26 + 8, 2 ** 26 + 3: 2 ** 26, 12345: 12345}
    for x, y in want.items():
        assert scheme.mma_fp32_model(x) == y * u, x


def test_apriori_bound_is_nearly_attained():
    """The closed-form bound sum_h (|b|/mu + |a|/nu + 1/(mu nu)) (from eq. def:A'/def:B',
    P:157-161) is attained up to ~1 %: positive entries whose scaled values have
    fractional part 1 - 2^-7 lose almost a whole unit to each truncation.  With fixed
    exponents (mu = 2^30, nu = 2^31) the exact error |C'/(mu nu) - AB| must lie in
    [0.98, 1] x bound: a bound off by a factor (or a dropped term) fails one side."""
    from oracle import exact
    k, N = 6, 12
    d = Fraction(127, 128)
    A = np.array([[float((Fraction(2 ** 45 + 17 * h) + d) / 2 ** 30) for h in range(k)]])
    B = np.array([[float((Fraction(2 ** 44 + 29 * h) + d) / 2 ** 31)] for h in range(k)])
    r = scheme.dgemm(A, B, N, e_mu=[30], e_nu=[31])
    Cp = Fraction(int(r.extra["Cprime"][0, 0]), 2 ** 61)
    ABx = sum(Fraction(float(A[0, h])) * Fraction(float(B[h, 0])) for h in range(k))
    err = abs(Cp - ABx)
    bnd = exact.apriori_bound(A, B, [30], [31])[0, 0]
    assert 0.98 * bnd <= float(err) <= bnd * (1 + 2 ** -40)
