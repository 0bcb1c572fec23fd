"""Pins for oracle.scheme / oracle.exact: worked examples, brute force, closed forms,
the certified condition and exactness identities.  All CPU (-m "not gpu")."""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact, fp8, fp32, models, moduli as mod, scheme
from synth import gen_host


# ------------------------------------------------------------------ digits / modprod

def test_digit_examples(spec):
    for p, r, d1, d2 in spec["digits_square"]["cases"]:
        assert scheme.digits_square(r, math.isqrt(p)) == (d1, d2)
    for r, d1, d2, d3 in spec["digits_karatsuba"]["cases"]:
        assert scheme.digits_karatsuba(r) == (d1, d2, d3)


def test_digits_exhaustive(facts):
    """Every residue of every hybrid modulus: reconstruction s*D1 + D2 = r and
    |D| <= 16, so each digit is an exact E4M3 integer."""
    dmax = facts["exactness_window"]["digit_max"]
    # hybrid moduli and the Karatsuba-only family (513, 512, ...: |r| <= 256, eq. limit1)
    for p in sorted(set(mod.hybrid_moduli(33)) | set(mod.karatsuba_moduli(33)), reverse=True):
        lo, hi = -(p // 2), (p + 1) // 2 - 1
        for r in range(lo, hi + 1):
            if mod.is_square(p):
                s = math.isqrt(p)
                d1, d2 = scheme.digits_square(r, s)
                assert s * d1 + d2 == r
                assert max(abs(d1), abs(d2)) <= dmax
            else:
                d1, d2, d3 = scheme.digits_karatsuba(r)
                assert 16 * d1 + d2 == r and d3 == d1 + d2
                assert max(abs(d1), abs(d2), abs(d3)) <= dmax
            for d in ((d1, d2) if mod.is_square(p) else (d1, d2, d3)):
                assert fp8.decode(fp8.encode_int(d)) == d


def test_exactness_window(facts):
    """k 2^4 2^4 <= 2^24 for k <= 2^16 (eq. error-free-FP8-matmult): the extreme sum
    is still a binary32 integer, and one more term would not be."""
    k = facts["exactness_window"]["k_max"]
    s = k * 16 * 16
    assert s == 2 ** 24 and float(np.float32(s)) == s
    assert float(np.float32(s + 1)) != s + 1


def test_modprod_examples(spec):
    e = spec["modprod_square"]
    p, a, b = e["p"], e["a"], e["b"]
    s = math.isqrt(p)
    Ad = [np.array([[x]]) for x in scheme.digits_square(a, s)]
    Bd = [np.array([[x]]) for x in scheme.digits_square(b, s)]
    assert scheme.modprod_square_digits(Ad, Bd, p)[0, 0] == e["c"] == mod.smod(a * b, p)
    e = spec["modprod_karatsuba"]
    p, a, b = e["p"], e["a"], e["b"]
    Ad = [np.array([[x]]) for x in scheme.digits_karatsuba(a)]
    Bd = [np.array([[x]]) for x in scheme.digits_karatsuba(b)]
    assert scheme.modprod_karatsuba_digits(Ad, Bd, p)[0, 0] == e["c"] == mod.smod(a * b, p)


def test_digit_route_equals_definition():
    """The FP8 digit route of Sec. III-B/C/D equals mod(A'_l B'_l, p_l) computed from
    the definition, for every modulus of the N=20 hybrid set (random residues)."""
    rng = np.random.default_rng(3)
    for p in mod.hybrid_moduli(20) + mod.karatsuba_moduli(4):
        for (m, k, n) in [(4, 37, 5), (3, 512, 2)]:
            lo, hi = -(p // 2), (p + 1) // 2 - 1
            Ar = rng.integers(lo, hi + 1, size=(m, k))
            Br = rng.integers(lo, hi + 1, size=(k, n))
            Ar[0, :] = hi            # extremes
            Br[:, 0] = lo
            want = scheme.modprod_direct(Ar, Br.T, p)
            Ad = scheme.digit_planes(Ar, p)
            Bd = scheme.digit_planes(Br, p)
            if mod.is_square(p):
                got = scheme.modprod_square_digits(Ad, Bd, p)
            else:
                got = scheme.modprod_karatsuba_digits(Ad, Bd, p)
            assert np.array_equal(got, want), p
            # brute force (pure Python) on the first entry
            bf = mod.smod(sum(int(Ar[0, h]) * int(Br[h, 0]) for h in range(k)), p)
            assert want[0, 0] == bf


# ------------------------------------------------------------------ scaling

def test_scaling_offset_example(spec):
    e = spec["scaling_offset"]
    t = scheme.offset_from_cbar(Fraction(e["cbar"]), Fraction(e["Pp"]), mod.delta())
    assert t == e["t"]
    # max c-bar = 1 -> offset int(P')
    assert scheme.offset_from_cbar(Fraction(1), Fraction(55), mod.delta()) == 55


def test_safety_factor_dominates_paper_factor():
    """f_k >= the paper's RU32(1 + (k+1) 2^-24) and >= the exact (1 - k 2^-24)^-1."""
    for k in [1, 2, 100, 4096, 4097, 8192, 16384, 65535, 65536]:
        f = scheme.safety_factor(k)
        paper = fp32.round_up(1 + Fraction(k + 1, 2 ** 24))
        assert f >= paper
        assert f >= Fraction(1) / (1 - Fraction(k, 2 ** 24))
        assert f >= Fraction(1) / (1 - Fraction(k, 2 ** 23))
    # the paper's factor is below the true (1 - k u)^-1 for k > 4096 (reading R5)
    k = 16384
    assert 1 + Fraction(k + 1, 2 ** 24) < Fraction(1) / (1 - Fraction(k, 2 ** 24))


def test_prescale_examples():
    # row max 3.7 -> ufp 2 -> mu' = 2^6; row max exactly 2^t -> scaled max 128
    e, codes = scheme.prescale_rows(np.array([[3.7, -1.0, 0.0]]))
    assert e == [6] and codes[0, 2] == 0
    e, codes = scheme.prescale_rows(np.array([[-2.0 ** 5, 1.0]]))
    assert e == [2] and fp8.decode(int(codes[0, 0])) == 128
    e, codes = scheme.prescale_rows(np.zeros((1, 4)))
    assert e == [0] and not codes.any()
    # scaled values stay < 2^8 (no overflow) and RU is an upper bound
    X = gen_host(6, 50, "phi", phi=4.0, seed=9, order="C")
    e, codes = scheme.prescale_rows(X)
    for r in range(6):
        for h in range(50):
            v = fp8.decode(int(codes[r, h]))
            y = abs(Fraction(float(X[r, h]))) * Fraction(2) ** e[r]
            assert y < 256 and v >= y and v <= 256


def test_prescale_fast_equals_reference():
    X = gen_host(5, 300, "phi", phi=4.0, seed=4, order="C")
    X[1, :] = 0.0
    X[2, 7] = 1e-300            # forces the tiny-value path
    X[3, :] *= 1e200
    e1, c1 = scheme.prescale_rows(X)
    e2, c2 = scheme.prescale_rows_fast(X)
    assert e1 == e2 and np.array_equal(c1, c2)


def test_to_integral_examples(spec):
    for x, e, want in spec["to_integral"]["cases"]:
        assert scheme.to_integral_row(np.array([x]), e) == [want]


def test_inverse_scale_examples(spec):
    for c, emu, enu, want in spec["inverse_scale"]["cases"]:
        Cp = np.empty((1, 1), dtype=object)
        Cp[0, 0] = c
        assert scheme.inverse_scale(Cp, [emu], [enu])[0, 0] == want


def test_residue_of_big(spec):
    e = spec["residue_of_big"]
    x = float(2 ** e["x_log2"])
    a = scheme.to_integral_row(np.array([x]), 0)[0]
    assert mod.smod(a, e["p"]) == e["r"]


# ------------------------------------------------------------------ exact references

def test_exact_dot_vs_fraction():
    A = gen_host(3, 40, "phi", phi=2.0, seed=1, order="C")
    B = gen_host(40, 4, "phi", phi=2.0, seed=2, order="C")
    F = exact.exact_gemm_fraction(A, B)
    E = exact.exact_entries(A, B, range(3), range(4))
    for i in range(3):
        for j in range(4):
            assert E[i, j] == float(F[i, j])
    # catastrophic cancellation
    a = np.array([1.0, 1.0])
    b = np.array([1.0, -(1.0 - 2.0 ** -52)])
    assert exact.exact_dot(a, b) == 2.0 ** -52


# ------------------------------------------------------------------ end to end

def _certified(res, A, B):
    """The condition 2 sum_h |a'_ih||b'_hj| < P, exactly in Python ints."""
    Aint, BintT, P = res.extra["Aint"], res.extra["BintT"], res.plan.P
    m, n = Aint.shape[0], BintT.shape[0]
    for i in range(m):
        ai = [abs(int(v)) for v in Aint[i]]
        for j in range(n):
            s = sum(x * abs(int(y)) for x, y in zip(ai, BintT[j]))
            if not 2 * s < P:
                return False
    return True


def test_identity_gives_identity(spec):
    for N in [6, 12]:
        I = np.eye(8)
        r = scheme.dgemm(I, I, N)
        assert np.array_equal(r.C, I)


def test_integer_inputs_exact():
    """Integers in [-2^20, 2^20], m=n=16, k=64, N=12 -> the exact product."""
    for seed in range(3):
        A = gen_host(16, 64, "int", seed=seed, order="C")
        B = gen_host(64, 16, "int", seed=100 + seed, order="C")
        r = scheme.dgemm(A, B, 12)
        want = (A.astype(object).dot(B.astype(object))).astype(np.float64)
        assert np.array_equal(r.C, want)


@pytest.mark.parametrize("N,phi", [(14, 0.0), (12, 1.0), (13, 4.0), (6, 0.5)])
def test_small_end_to_end_vs_brute_force(N, phi):
    """64^3-class check of the whole oracle against exact rational DGEMM:
    certified condition, C' = A'B' exactly (CRT identity), residues consistent with
    C', and |C - AB| within the closed-form a-priori bound."""
    m, k, n = 12, 40, 10
    A = gen_host(m, k, "phi", phi=phi, seed=11, order="C")
    B = gen_host(k, n, "phi", phi=phi, seed=12, order="C")
    A[3, :] = 0.0                       # zero row
    B[:, 2] = 0.0                       # zero column
    r = scheme.dgemm(A, B, N)
    assert _certified(r, A, B)
    exactP = r.extra["Aint"].dot(r.extra["BintT"].T)
    for i in range(m):
        for j in range(n):
            assert int(r.extra["Cprime"][i, j]) == int(exactP[i, j])
            for l, p in enumerate(r.plan.moduli):
                assert (int(exactP[i, j]) - int(r.residues[l][i, j])) % p == 0
    F = exact.exact_gemm_fraction(A, B)
    bound = exact.apriori_bound(A, B, r.e_mu, r.e_nu)
    for i in range(m):
        for j in range(n):
            err = abs(Fraction(float(r.C[i, j])) - F[i, j])
            allowed = Fraction(2 * bound[i, j]) + abs(F[i, j]) * Fraction(2, 2 ** 53)
            assert err <= allowed
    assert not r.C[3, :].any() and not r.C[:, 2].any()
    assert r.e_mu[3] == 0 and r.e_nu[2] == 0


def test_error_drops_with_moduli():
    """Each added modulus raises mu, nu by ~log2 sqrt(p) ~ 4.5 bits:
    normwise error vs the exact product falls monotonically until the binary64
    output-rounding floor."""
    A = gen_host(6, 300, "phi", phi=1.0, seed=21, order="C")
    B = gen_host(300, 6, "phi", phi=1.0, seed=22, order="C")
    E = exact.exact_entries(A, B, range(6), range(6))
    errs = []
    for N in [6, 7, 8, 9, 10, 12, 14]:
        r = scheme.dgemm(A, B, N)
        errs.append(np.linalg.norm(r.C - E) / np.linalg.norm(E))
    for a, b in zip(errs, errs[1:]):
        assert b <= a * 1.01 or b < 1e-16
    # 6 -> 7 moduli: about one 9-bit modulus more in P, ~4.5 bits more per side
    assert errs[1] < errs[0] / 8
    assert errs[-1] < 2e-16


def test_alpha_beta():
    A = gen_host(4, 16, "phi", phi=1.0, seed=31, order="C")
    B = gen_host(16, 5, "phi", phi=1.0, seed=32, order="C")
    C0 = gen_host(4, 5, "uniform", seed=33, order="C")
    r1 = scheme.dgemm(A, B, 12)
    r2 = scheme.dgemm(A, B, 12, alpha=-2.0, beta=0.5, C=C0)
    # alpha = -2 is exact scaling; beta*C0 is exact (power of two); one rounding of the sum
    want = np.array([[float(Fraction(-2) * Fraction(float(r1.C[i, j])) + Fraction(0.5) * Fraction(float(C0[i, j])))
                      for j in range(5)] for i in range(4)])
    assert np.array_equal(r2.C, want)
    r3 = scheme.dgemm(A, B, 12, alpha=2.0, beta=0.0, C=np.full((4, 5), np.nan))
    assert np.array_equal(r3.C, 2.0 * r1.C)


def test_entries_match_full_oracle():
    """The sampled-entry path (used at full sizes) equals the full oracle."""
    A = gen_host(9, 70, "phi", phi=2.0, seed=41, order="C")
    B = gen_host(70, 8, "phi", phi=2.0, seed=42, order="C")
    r = scheme.dgemm(A, B, 13)
    I, J = [0, 4, 8], [1, 7]
    eA, emu, _ = scheme.row_exponents(A, I, B.T, 13)
    eB, enu, _ = scheme.row_exponents(B.T, J, A, 13)
    assert emu == [r.e_mu[i] for i in I] and enu == [r.e_nu[j] for j in J]
    assert eA == [r.e_prime_A[i] for i in I]
    res, C = scheme.entries(A, B, 13, I, J, emu, enu)
    for a, i in enumerate(I):
        for b, j in enumerate(J):
            assert C[a, b] == r.C[i, j]
            for l in range(13):
                assert res[l, a, b] == r.residues[l][i, j]


# ------------------------------------------------------------------ fast mode (NEXT-1)

def test_fast_offset_definition():
    """t = max{t : 2^(2t) S <= H}: bracketing check, including exact powers of two."""
    from fractions import Fraction as F
    plan, _, _ = scheme.plan_constants(12)
    H = scheme.fast_H(plan)
    assert H <= F(plan.P - 1, 2) < H * (1 + F(1, 2 ** 52))
    for S in [F(1), F(3, 7), F(2) ** -18, F(225, 2 ** 18), F(2) ** 38, H, H / 4, H * 4 + 1]:
        t = scheme.fast_offset(S, H)
        assert F(2) ** (2 * t) * S <= H < F(2) ** (2 * (t + 1)) * S
    # S = H / 4 exactly -> t = 1 (boundary inclusive)
    assert scheme.fast_offset(H / 4, H) == 1


def test_fast_H_small_P():
    """N = 2: P = 1089 * 1024, (P-1)/2 is exactly representable."""
    from fractions import Fraction as F
    plan, _, _ = scheme.plan_constants(2)
    assert scheme.fast_H(plan) == F(1089 * 1024 - 1, 2)


@pytest.mark.parametrize("phi", [0.0, 2.0])
def test_fast_mode_certified_and_less_accurate(phi):
    """Fast mode satisfies the condition 2 sum|a'||b'| < P exactly (Cauchy-Schwarz),
    and its error is >= accurate mode's at equal N."""
    m, k, n = 10, 60, 9
    A = gen_host(m, k, "phi", phi=phi, seed=71, order="C")
    B = gen_host(k, n, "phi", phi=phi, seed=72, order="C")
    rf = scheme.dgemm(A, B, 12, mode="fast")
    ra = scheme.dgemm(A, B, 12)
    assert _certified(rf, A, B)
    exactP = rf.extra["Aint"].dot(rf.extra["BintT"].T)
    assert all(int(rf.extra["Cprime"][i, j]) == int(exactP[i, j]) for i in range(m) for j in range(n))
    # the bound is Cauchy-Schwarz over the FP8 upper bounds: recompute S_i by brute force
    for i in range(m):
        Si = sum(Fraction(fp8.decode(int(c))) ** 2 for c in rf.Abar[i])
        H = scheme.fast_H(rf.plan)
        t = rf.e_mu[i] - rf.e_prime_A[i]
        assert Fraction(4) ** t * Si <= H < Fraction(4) ** (t + 1) * Si
    F = exact.exact_gemm_fraction(A, B)
    ex = np.array([[float(F[i, j]) for j in range(n)] for i in range(m)])
    ef = np.linalg.norm(rf.C - ex) / np.linalg.norm(ex)
    ea = np.linalg.norm(ra.C - ex) / np.linalg.norm(ex)
    assert ea <= ef * 1.0000001 or ef < 1e-17


# ------------------------------------------------------------------ Karatsuba-only family (NEXT-4)

def test_karatsuba_family_limits(facts):
    """eq. limit1: every Karatsuba-family residue satisfies |r| <= 256 (p <= 513),
    the Karatsuba digits of +-256 are the extreme +-16, and no family member up to
    N = 33 is a square (so every modulus takes the 3-digit route, 3N GEMMs)."""
    ps = mod.karatsuba_moduli(33)
    assert max(ps) == 513 and not any(mod.is_square(p) for p in ps)
    for p in ps:
        assert p // 2 <= 256 and (p + 1) // 2 - 1 <= 256
    assert scheme.digits_karatsuba(256) == (16, 0, 16)
    assert scheme.digits_karatsuba(-256) == (-16, 0, -16)
    plan, _, _ = scheme.plan_constants(13, "karatsuba")
    assert plan.moduli == tuple(ps[:13])
    assert plan.P // 2 > 2 ** 115


@pytest.mark.parametrize("N,phi", [(13, 1.0), (4, 0.5)])
def test_karatsuba_family_end_to_end(N, phi):
    """The whole oracle with the Karatsuba-only moduli: certified condition, C' = A'B'
    exactly, residues consistent with C', C within the a-priori bound (as for the
    hybrid family), and the FP8 digit route of every modulus equals the definition."""
    m, k, n = 9, 33, 8
    A = gen_host(m, k, "phi", phi=phi, seed=81, order="C")
    B = gen_host(k, n, "phi", phi=phi, seed=82, order="C")
    r = scheme.dgemm(A, B, N, family="karatsuba", want_digits=True)
    assert r.plan.moduli == tuple(mod.karatsuba_moduli(N))
    assert _certified(r, A, B)
    exactP = r.extra["Aint"].dot(r.extra["BintT"].T)
    for i in range(m):
        for j in range(n):
            assert int(r.extra["Cprime"][i, j]) == int(exactP[i, j])
            for l, p in enumerate(r.plan.moduli):
                assert (int(exactP[i, j]) - int(r.residues[l][i, j])) % p == 0
    for l, p in enumerate(r.plan.moduli):
        Ad, Bd = r.extra["digits"][l]
        assert len(Ad) == 3 and len(Bd) == 3
        assert np.array_equal(scheme.modprod_karatsuba_digits(Ad, [b.T for b in Bd], p), r.residues[l])
    F = exact.exact_gemm_fraction(A, B)
    bound = exact.apriori_bound(A, B, r.e_mu, r.e_nu)
    for i in range(m):
        for j in range(n):
            err = abs(Fraction(float(r.C[i, j])) - F[i, j])
            assert err <= Fraction(2 * bound[i, j]) + abs(F[i, j]) * Fraction(2, 2 ** 53)


def test_karatsuba_13_matches_hybrid_12_accuracy():
    """the Karatsuba family needs N >= 13 where the hybrid family
    needs N >= 12 for FP64-level accuracy (P/2 > 2^115 vs 2^110).  At equal N the hybrid
    family (larger P) is at least as accurate; Karatsuba N = 13 is at least as accurate as
    hybrid N = 12."""
    A = gen_host(6, 300, "phi", phi=1.0, seed=91, order="C")
    B = gen_host(300, 6, "phi", phi=1.0, seed=92, order="C")
    E = exact.exact_entries(A, B, range(6), range(6))
    err = lambda r: np.linalg.norm(r.C - E) / np.linalg.norm(E)
    eh = {N: err(scheme.dgemm(A, B, N)) for N in (10, 11, 12)}
    ek = {N: err(scheme.dgemm(A, B, N, family="karatsuba")) for N in (10, 11, 12, 13)}
    for N in (10, 11, 12):
        assert mod.crt_plan(mod.karatsuba_moduli(N)).P < mod.crt_plan(mod.hybrid_moduli(N)).P
        assert eh[N] <= ek[N]
    assert ek[13] <= eh[12]
    assert ek[11] < ek[10] / 8 and ek[12] < ek[11] / 8     # ~4.5 bits per modulus
