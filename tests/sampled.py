"""Sampled parity at sizes where the full oracle is too slow (helpers for the -m gpu
tests; host-side only, imports the oracle, never the CUDA path).

``tile_cover`` picks one row per 256-row tile of C and one column per 256-column tile,
so the sampled I x J grid touches EVERY output tile of the residue GEMM exactly once --
hence every persistent unit's every tile, including each unit's last tile (the one whose
CRT runs deferred in the fused-CRT schedule).  Within its tile the row offset cycles
through both CTAs of a CTA pair (rows 0-127 / 128-255) and the four TMEM lane quadrants
(32-row groups, one per epilogue warp); the column offset cycles through both 128-column
epilogue halves.

``check_sampled`` compares the GPU's exponents, residues and C of the sampled entries
with the oracle's.  Exponents may differ from the oracle's own only inside the R6
rounding window (reading R13); such a row / column is validated instead: its offset must
lie in the window, the certified condition 2 sum_h |a'_ih||b'_hj| < P must
hold for that row against ALL columns (GPU exponents, a rigorous binary64 upper bound),
and its entries are then recomputed by the oracle with the GPU's exponents and must be
bit-exact.  Every sampled residue and C entry is compared bit for bit.
"""
from fractions import Fraction

import numpy as np

from oracle import exact, int8, scheme


def tile_cover(extent: int, tile: int = 256, seed: int = 0):
    rng = np.random.default_rng(seed + extent)
    out = []
    for t in range((extent + tile - 1) // tile):
        half = (t % 2) * 128
        quad = ((t // 2) % 4) * 32
        off = half + quad + int(rng.integers(0, 32))
        r = t * tile + off
        if r >= extent:                      # ragged last tile
            r = extent - 1 - int(rng.integers(0, min(32, extent - t * tile)))
        out.append(r)
    return out


def col_cover(extent: int, tile: int = 256, seed: int = 1):
    rng = np.random.default_rng(seed + 3 * extent)
    out = []
    for t in range((extent + tile - 1) // tile):
        off = (t % 2) * 128 + int(rng.integers(0, 128))
        c = t * tile + off
        if c >= extent:
            c = extent - 1 - int(rng.integers(0, min(128, extent - t * tile)))
        out.append(c)
    return out


def _certify_rows(X, rows, e_rows, Y_T, e_all, P):
    """2 sum_h |x'_rh||y'_jh| < P for every j, with x' = trunc(2^e x) (rows of X) and
    y' = trunc(2^e_all Y_T): binary64 dot of exact-ish magnitudes, bounded above by
    (1 + (k + 3) 2^-52) (each |x'| and |y'| rounds by <= 2^-53 relative, the dot by
    <= k 2^-53)."""
    k = X.shape[1]
    Yi = np.abs(np.trunc(np.ldexp(Y_T, np.asarray(e_all, dtype=np.int64)[:, None])))
    for r, e in zip(rows, e_rows):
        xr = np.abs(np.trunc(np.ldexp(X[r], int(e))))
        s = Yi @ xr
        ub = s.max() * (1.0 + (k + 3) * 2.0 ** -52)
        assert 2.0 * ub < float(P), ("certified condition", r)


def _window_ok(R, e_gpu, e_prime, k, N, family):
    plan, Pp, dlt = scheme.plan_constants(N, family)
    lo = scheme.scaling_offset(R * (1 - Fraction(k, 2 ** 23)), k, Pp, dlt)
    hi = scheme.scaling_offset(R * (1 + Fraction(1, 2 ** 23)), k, Pp, dlt)
    return hi <= e_gpu - e_prime <= lo


def check_sampled(A, B, N, I, J, gpu, family="hybrid", mode="accurate", accuracy=True):
    """gpu: dict with 'e_mu' / 'e_nu' (FULL vectors), 'res' [N][|I|][|J|] (optional) and
    'C' [|I|][|J|].  A (m x k), B (k x n) host float64.  Returns the normwise error of the
    sampled C against the exact product (if accuracy)."""
    k = A.shape[1]
    BT = np.ascontiguousarray(B.T)
    gmu = np.asarray(gpu["e_mu"])[I].tolist()
    gnu = np.asarray(gpu["e_nu"])[J].tolist()
    moduli = int8.plan(N).moduli if family == "int8" else None
    if family == "int8":
        _, emu = int8.row_exponents(A, I, BT, N, mode)
        _, enu = int8.row_exponents(BT, J, A, N, mode)
        assert gmu == emu and gnu == enu          # R16: exact integer bound, no window
    elif mode == "fast":
        plan, _, _ = scheme.plan_constants(N, family)
        eA, cA = scheme.prescale_rows_fast(np.ascontiguousarray(A[I]))
        eB, cB = scheme.prescale_rows_fast(np.ascontiguousarray(BT[J]))
        emu = scheme.fast_exponents(eA, cA, plan, [not np.any(A[i]) for i in I])
        enu = scheme.fast_exponents(eB, cB, plan, [not np.any(BT[j]) for j in J])
        assert gmu == emu and gnu == enu          # R15: decided in exact integers
    else:
        eA, emu, RA = scheme.row_exponents(A, I, BT, N, family)
        eB, enu, RB = scheme.row_exponents(BT, J, A, N, family)
        bad_r = [a for a in range(len(I)) if gmu[a] != emu[a]]
        bad_c = [b for b in range(len(J)) if gnu[b] != enu[b]]
        assert len(bad_r) <= max(1, len(I) // 32) and len(bad_c) <= max(1, len(J) // 32)
        plan, _, _ = scheme.plan_constants(N, family)
        for a in bad_r:
            assert _window_ok(RA[a], gmu[a], eA[a], k, N, family), ("row window", I[a])
        for b in bad_c:
            assert _window_ok(RB[b], gnu[b], eB[b], k, N, family), ("col window", J[b])
        if bad_r:
            _certify_rows(A, [I[a] for a in bad_r], [gmu[a] for a in bad_r], BT, gpu["e_nu"], plan.P)
        if bad_c:
            _certify_rows(BT, [J[b] for b in bad_c], [gnu[b] for b in bad_c], A, gpu["e_mu"], plan.P)
    # given the exponents, residues and C are unique (R13): bit-exact against the oracle
    res, Cref = scheme.entries(A, B, N, I, J, gmu, gnu, family, moduli=moduli)
    if gpu.get("res") is not None:
        assert np.array_equal(np.asarray(gpu["res"]), res)
    assert np.array_equal(np.asarray(gpu["C"]), Cref)
    if not accuracy:
        return None
    ex = exact.exact_entries(A, B, I, J)
    bound = exact.apriori_bound(A[I], B[:, J], gmu, gnu)
    assert np.all(np.abs(Cref - ex) <= 2 * bound + np.abs(ex) * 2.0 ** -52)
    return float(np.linalg.norm(Cref - ex) / np.linalg.norm(ex))
