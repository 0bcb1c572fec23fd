"""Exact references for the product AB itself (not the scheme).

* ``exact_gemm_fraction``: brute-force exact rational DGEMM (tiny sizes).
* ``exact_dot``: the exact dot product of two binary64 vectors, rounded once to
  nearest binary64.  Each product a*b is split exactly into p + e with Dekker's
  TwoProduct (Veltkamp splitting, no FMA needed; exact barring over/underflow,
  asserted), then ``math.fsum`` returns the correctly rounded value of the exact
  sum of all 2k terms.  Cross-checked against ``exact_gemm_fraction`` in tests.
* ``apriori_bound``: the closed-form error bound of the scheme derived from
  eq. def:A' / def:B' and P:186: with |mu_i a_ih - a'_ih| < 1 and
  |b_hj nu_j - b'_hj| < 1 and C' = A'B' exactly (condition),
      |C'_ij/(mu_i nu_j) - (AB)_ij| <= sum_h (|b_hj|/mu_i + |a_ih|/nu_j + 1/(mu_i nu_j)).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math
from fractions import Fraction

import numpy as np

_SPLIT = 134217729.0  # 2^27 + 1


def exact_gemm_fraction(A: np.ndarray, B: np.ndarray):
    m, k = A.shape
    _, n = B.shape
    out = np.empty((m, n), dtype=object)
    Af = [[Fraction(float(v)) for v in row] for row in A]
    Bf = [[Fraction(float(B[h, j])) for h in range(k)] for j in range(n)]
    for i in range(m):
        for j in range(n):
            out[i, j] = sum((a * b for a, b in zip(Af[i], Bf[j])), Fraction(0))
    return out


def _split(x: np.ndarray):
    c = _SPLIT * x
    hi = c - (c - x)
    return hi, x - hi


def exact_dot(a: np.ndarray, b: np.ndarray) -> float:
    """RN64(sum_h a_h b_h) exactly (Dekker TwoProduct + fsum)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    p = a * b
    nz = p != 0
    if np.any(nz):
        ap = np.abs(p[nz])
        # TwoProduct is exact when no intermediate over/underflows
        assert ap.max() < 2.0 ** 960 and ap.min() > 2.0 ** -960, "exact_dot range"
        assert np.abs(a).max() < 2.0 ** 995 and np.abs(b).max() < 2.0 ** 995
    ah, al = _split(a)
    bh, bl = _split(b)
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    return math.fsum(np.concatenate([p, e]).tolist())


def exact_entries(A: np.ndarray, B: np.ndarray, I, J) -> np.ndarray:
    out = np.zeros((len(I), len(J)))
    for a, i in enumerate(I):
        for b, j in enumerate(J):
            out[a, b] = exact_dot(A[i, :], B[:, j])
    return out


def apriori_bound(A: np.ndarray, B: np.ndarray, e_mu, e_nu) -> np.ndarray:
    """sum_h (|b_hj| 2^-e_mu_i + |a_ih| 2^-e_nu_j + 2^-(e_mu_i+e_nu_j)), as floats
    (the bound is compared with a factor-2 allowance for its own rounding)."""
    m, k = A.shape
    n = B.shape[1]
    sa = np.abs(A).sum(axis=1)
    sb = np.abs(B).sum(axis=0)
    out = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            out[i, j] = (sb[j] * 2.0 ** (-e_mu[i]) + sa[i] * 2.0 ** (-e_nu[j])
                         + k * 2.0 ** (-(e_mu[i] + e_nu[j])))
    return out
