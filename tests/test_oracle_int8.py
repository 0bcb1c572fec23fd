"""Pins for oracle.int8 (INT8 Ozaki-II; reading R16): prescale bounds,
exactness windows, the certified condition checked exactly, the CRT identity C' = A'B',
brute-force exact rational DGEMM, and the error falling with N.  All CPU."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, int8, moduli as mod, scheme
from synth import gen_host


def _certified(res):
    Aint, BintT, P = res.extra["Aint"], res.extra["BintT"], res.plan.P
    for i in range(Aint.shape[0]):
        ai = [abs(int(v)) for v in Aint[i]]
        for j in range(BintT.shape[0]):
            if not 2 * sum(x * abs(int(y)) for x, y in zip(ai, BintT[j])) < P:
                return False
    return True


def test_prescale_bounds():
    X = gen_host(7, 90, "phi", phi=4.0, seed=3, order="C")
    X[2, :] = 0.0
    X[4, 5] = 1e-300
    e, bars = int8.prescale_rows(X)
    assert e[2] == 0 and not bars[2].any()
    for r in range(7):
        if r == 2:
            continue
        mx = max(abs(Fraction(float(v))) for v in X[r]) * Fraction(2) ** e[r]
        assert 64 <= mx < 128                           # 2^6 <= max scaled < 2^7
        for h in range(90):
            y = abs(Fraction(float(X[r, h]))) * Fraction(2) ** e[r]
            b = int(bars[r, h])
            assert b >= y and b - 1 < y and b <= 128    # ceil: the smallest integer >= y
    assert bars[4, 5] == 1                              # tiny nonzero -> 1


def test_residue_and_product_windows():
    """|mod(x, p)| <= 128 for every INT8 modulus (one INT8 operand) and
    k 128^2 <= 2^30 for k <= 2^16: every INT32 partial sum is exact."""
    for p in mod.int8_moduli(33):
        assert p <= 256
        lo, hi = -(p // 2), (p + 1) // 2 - 1
        assert -128 <= lo and hi <= 127
        assert mod.smod(lo, p) == lo and mod.smod(hi, p) == hi
    assert 2 ** 16 * 128 * 128 == 2 ** 30 < 2 ** 31


@pytest.mark.parametrize("mode", ["accurate", "fast"])
@pytest.mark.parametrize("phi,N", [(0.0, 14), (2.0, 14), (4.0, 16), (1.0, 6)])
def test_certified_and_crt_identity(mode, phi, N):
    A = gen_host(9, 70, "phi", phi=phi, seed=11, order="C")
    B = gen_host(70, 8, "phi", phi=phi, seed=12, order="C")
    r = int8.dgemm(A, B, N, mode=mode)
    assert _certified(r)
    exactP = r.extra["Aint"].dot(r.extra["BintT"].T)
    assert all(int(r.extra["Cprime"][i, j]) == int(exactP[i, j]) for i in range(9) for j in range(8))
    # the exponent is the largest t with 2^(2t) U <= H (R16): bracket it
    H = scheme.fast_H(r.plan)
    for i in range(9):
        t = r.e_mu[i] - r.e_prime_A[i]
        U = Fraction(r.R[i])
        assert Fraction(4) ** t * U <= H < Fraction(4) ** (t + 1) * U


def test_bound_is_exact_product():
    A = gen_host(6, 40, "phi", phi=1.0, seed=13, order="C")
    B = gen_host(40, 5, "phi", phi=1.0, seed=14, order="C")
    _, Ab = int8.prescale_rows(A)
    _, BbT = int8.prescale_rows(B.T.copy())
    R, S, Cb = int8.bound_row_col_max(Ab, BbT)
    for i in range(6):
        for j in range(5):
            assert Cb[i, j] == sum(int(Ab[i, h]) * int(BbT[j, h]) for h in range(40))
    assert R == [max(int(Cb[i, j]) for j in range(5)) for i in range(6)]
    assert S == [max(int(Cb[i, j]) for i in range(6)) for j in range(5)]


def test_brute_force_rational_and_apriori_bound():
    A = gen_host(5, 24, "phi", phi=2.0, seed=15, order="C")
    B = gen_host(24, 6, "phi", phi=2.0, seed=16, order="C")
    r = int8.dgemm(A, B, 14)
    F = exact.exact_gemm_fraction(A, B)
    bound = exact.apriori_bound(A, B, r.e_mu, r.e_nu)
    for i in range(5):
        for j in range(6):
            assert abs(Fraction(float(r.C[i, j])) - F[i, j]) <= 2 * Fraction(bound[i, j]) + \
                abs(F[i, j]) * Fraction(1, 2 ** 52)


def test_identity_and_integers_exact():
    I = np.eye(12)
    X = gen_host(12, 12, "uniform", seed=17, order="C")
    assert np.array_equal(int8.dgemm(I, X, 14).C, X)
    Ai = gen_host(6, 30, "int", seed=18, order="C")
    Bi = gen_host(30, 7, "int", seed=19, order="C")
    assert np.array_equal(int8.dgemm(Ai, Bi, 16).C, Ai @ Bi)


def test_error_falls_with_N():
    """Each INT8 modulus adds ~ log2 sqrt(p) ~ 4 bits to mu and nu (Table 2: N = 14 is
    the first FP64-level count)."""
    A = gen_host(8, 512, "phi", phi=1.0, seed=20, order="C")
    B = gen_host(512, 8, "phi", phi=1.0, seed=21, order="C")
    F = exact.exact_gemm_fraction(A, B)
    ex = np.array([[float(F[i, j]) for j in range(8)] for i in range(8)])
    errs = []
    for N in [10, 11, 12, 13, 14]:
        C = int8.dgemm(A, B, N).C
        errs.append(np.linalg.norm(C - ex) / np.linalg.norm(ex))
    for a, b in zip(errs, errs[1:]):
        assert b < a / 4 or b < 1e-16
    assert errs[-1] < 1e-15
