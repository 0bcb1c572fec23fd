"""The INT8 Ozaki-II DGEMM emulation (the paper's Sec. II baseline, Table 2's
INT8 rows P:463-471), step by step.

  1. prescale   e'_i = 6 - floor(log2 max_h |a_ih|), A-bar = ceil(|a| 2^e') in [0, 128]  (R16)
  2. bound      C-bar = A-bar B-bar, exact in INT32 (k 2^14 <= 2^30 for k <= 2^16)        (R16)
  3. exponents  log2 mu_i = e'_i + max{t : 2^(2t) R_i <= H}, H = RD64((P-1)/2)            (R16)
     (fast mode: R_i replaced by S_i = sum_h abar_ih^2, Cauchy-Schwarz, R15/R16)
  4. integers   A' = trunc(diag(mu) A), B' = trunc(B diag(nu))                             eq. def:A'
  5. residues   A'_l = mod(A', p_l), p_l from the INT8 list: |A'_l| <= 128
  6. products   C'_l = mod(A'_l B'_l, p_l) (one INT8 GEMM per modulus)              eq. CRTmatmul
  7. CRT        C' = mod(sum_l q_l P/p_l C'_l, P)                                           eq. CRT_finalreduction
  8. unscale    C = diag(mu)^-1 C' diag(nu)^-1                                              eq. inversescaling

Steps 4-8 are the shared Ozaki-II skeleton (``scheme.to_integral`` ... ``scheme.alpha_beta``);
only the moduli, the prescale and the exponent rule differ from the FP8 scheme.

Reading R16: this paper cites the INT8 accurate mode ("the upper bound
is estimated by matrix multiplication using INT8 MMA units") without giving its formulas.
With A-bar = ceil(2^e'|a|) the bound product is exact, so the split of the budget between
mu and nu needs no rounding compensation (no delta, no f_k): 2 sum_h |a'||b'| <=
2 2^(t_i + t_j) c-bar_ij <= 2 sqrt(2^(2t_i) R_i 2^(2t_j) S_j) <= 2H < P when each side
satisfies 2^(2t) R <= H.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import math
from fractions import Fraction

import numpy as np

from . import moduli as mod
from . import scheme


def plan(N: int):
    """CRT plan of the first N INT8 moduli (eq. p_list)."""
    if not 2 <= N <= 33:
        raise ValueError("INT8 moduli: N in [2, 33]")
    return mod.crt_plan(mod.int8_moduli(N))


def prescale_rows(X: np.ndarray):
    """e'_r = 6 - floor(log2 max_h |x_rh|) (zero row -> 0, R3) and the exact upper bounds
    Xbar_rh = ceil(|x_rh| 2^e'_r) in [0, 128] (max scaled value in [64, 128))."""
    rows, k = X.shape
    e_prime = []
    bars = np.zeros((rows, k), dtype=np.int64)
    for r in range(rows):
        row = X[r]
        mx = float(np.max(np.abs(row))) if k else 0.0
        if mx == 0.0:
            e_prime.append(0)
            continue
        e = 6 - scheme.ufp_exp(mx)
        e_prime.append(e)
        scale = Fraction(2) ** e
        for h in range(k):
            v = float(row[h])
            if v != 0.0:
                bars[r, h] = math.ceil(abs(Fraction(v)) * scale)
    return e_prime, bars


def bound_row_col_max(Abar: np.ndarray, Bbar_T: np.ndarray):
    """Exact C-bar = A-bar B-bar (integers) and its row / column maxima R, S."""
    Cb = scheme.exact_int_matmul(Abar, Bbar_T.T)
    m, n = Cb.shape
    R = [int(Cb[i].max()) if n else 0 for i in range(m)]
    S = [int(Cb[:, j].max()) if m else 0 for j in range(n)]
    return R, S, Cb


def exponents(e_prime, U, pl, row_zero):
    """log2 mu_r = e'_r + max{t : 2^(2t) U_r <= H} (R16); zero rows 0 (R3); U_r = 0 on a
    nonzero row (every product zero) keeps e'_r."""
    H = scheme.fast_H(pl)
    out = []
    for e, u, z in zip(e_prime, U, row_zero):
        if z:
            out.append(0)
        elif u == 0:
            out.append(int(e))
        else:
            out.append(int(e) + scheme.fast_offset(Fraction(u), H))
    return out


def dgemm(A: np.ndarray, B: np.ndarray, N: int, alpha: float = 1.0, beta: float = 0.0,
          C=None, mode: str = "accurate", e_mu=None, e_nu=None) -> scheme.Result:
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    if not (np.all(np.isfinite(A)) and np.all(np.isfinite(B))):
        raise ValueError("non-finite input (reading R12)")
    pl = plan(N)
    BT = B.T.copy()
    eA, Abar = prescale_rows(A)
    eB, BbarT = prescale_rows(BT)
    zA = [not np.any(A[i]) for i in range(m)]
    zB = [not np.any(BT[j]) for j in range(n)]
    if mode == "fast":
        R = [int(sum(int(v) ** 2 for v in row)) for row in Abar]
        S = [int(sum(int(v) ** 2 for v in row)) for row in BbarT]
    else:
        R, S, _ = bound_row_col_max(Abar, BbarT)
    if e_mu is None:
        e_mu = exponents(eA, R, pl, zA)
    if e_nu is None:
        e_nu = exponents(eB, S, pl, zB)
    Aint = scheme.to_integral(A, e_mu)
    BintT = scheme.to_integral(BT, e_nu)
    res = []
    for p in pl.moduli:
        res.append(scheme.modprod_direct(scheme.residues(Aint, p), scheme.residues(BintT, p), p))
    Cp = scheme.crt_combine(res, pl) if m and n else np.zeros((m, n), dtype=object)
    X = scheme.inverse_scale(Cp, e_mu, e_nu)
    if alpha != 1.0 or beta != 0.0:
        X = scheme.alpha_beta(X, alpha, beta, C)
    r = scheme.Result(X, eA, eB, Abar, BbarT, R, S, list(e_mu), list(e_nu), res, pl,
                      Fraction(0), Fraction(0), Fraction(1))
    r.extra["Cprime"] = Cp
    r.extra["Aint"] = Aint
    r.extra["BintT"] = BintT
    return r


def prescale_rows_fast(X: np.ndarray):
    """Vectorised prescale_rows (same definition; pinned equal in tests): ldexp by the
    row exponent is exact for normal results, and a nonzero entry whose scaled value
    underflows still gets the upper bound 1."""
    X = np.asarray(X, dtype=np.float64)
    rows, k = X.shape
    ax = np.abs(X)
    mx = ax.max(axis=1) if k else np.zeros(rows)
    e_prime = np.zeros(rows, dtype=np.int64)
    nz = mx > 0
    _, ex = np.frexp(mx[nz])
    e_prime[nz] = 6 - (ex - 1)
    y = np.ceil(np.ldexp(ax, np.broadcast_to(e_prime[:, None], ax.shape)))
    y = np.where((ax > 0) & (y == 0), 1.0, y)
    return e_prime.tolist(), y.astype(np.int64)


def row_exponents(X: np.ndarray, rows, Y_T: np.ndarray, N: int, mode: str = "accurate"):
    """e' and log2 mu for selected rows r of X against the full other operand Y_T
    (accurate mode: R_r = max_j (A-bar B-bar)_rj, exact; fast: S_r = sum_h abar_rh^2)."""
    pl = plan(N)
    rows = list(rows)
    e1, xb = prescale_rows_fast(np.ascontiguousarray(X[rows]))
    if mode == "fast":
        U = [int(sum(int(v) ** 2 for v in r)) for r in xb]
    else:
        _, yb = prescale_rows_fast(Y_T)
        assert X.shape[1] * 2 ** 14 < 2 ** 53
        prod = xb.astype(np.float64) @ yb.astype(np.float64).T      # exact integers
        U = [int(v) for v in np.rint(prod.max(axis=1))] if prod.size else [0] * len(rows)
    z = [not np.any(X[r]) for r in rows]
    return e1, exponents(e1, U, pl, z)
