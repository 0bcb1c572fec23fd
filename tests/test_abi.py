"""The C-ABI library loads, exports every symbol include/oz2.h declares, and its
host-only planner agrees with the oracle (no device needed, no compute calls)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "oz2.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(oz2_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def oz2mod():
    import paper_2603_10634_b200 as P
    P.lib()
    return P


def test_header_symbols_exported(oz2mod):
    names = _declared()
    assert "oz2_dgemm" in names and len(names) >= 10
    out = subprocess.run(["nm", "-D", "--defined-only", oz2mod.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (oz2_[a-z0-9_]+)", out))
    assert set(names) <= exported, set(names) - exported
    bound = {s[0] for s in oz2mod.SIGNATURES}
    assert set(names) == bound            # the binding covers exactly the header surface
    for n in names:
        assert hasattr(oz2mod.lib(), n)


def test_built_for_sm100a(oz2mod):
    out = subprocess.run(["cuobjdump", "--list-elf", oz2mod.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", oz2mod.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCQMMA" in sass          # tcgen05.mma kind::f8f6f4
    assert "UTMALDG" in sass          # TMA loads
    assert "LDTM" in sass             # tcgen05.ld
    assert "HMMA" not in sass and "QGMMA" not in sass


def test_version(oz2mod):
    assert "sm_100a" in oz2mod.oz2_version()


def test_moduli_match_oracle(oz2mod):
    from oracle import moduli as mod
    for N in [2, 6, 7, 12, 13, 14, 20, 33]:
        assert oz2mod.oz2_moduli(N) == mod.hybrid_moduli(N)


def test_plan_constants_match_oracle(oz2mod):
    from fractions import Fraction
    from oracle import fp32, models, moduli as mod, scheme
    for N in [2, 6, 12, 13, 14, 16, 20, 33]:
        for k in [1, 64, 4096, 8192, 16384, 65536]:
            info = oz2mod.oz2_plan_query(N, k)
            plan = mod.crt_plan(mod.hybrid_moduli(N))
            assert info.num_planes == models.M_N(N)
            assert info.num_squares == min(N, 6)
            assert Fraction(info.p_prime) == mod.p_prime(plan.P)
            assert Fraction(info.delta) == mod.delta()
            assert Fraction(info.f_k) == scheme.safety_factor(k)
            L = info.num_limbs
            assert 2 ** (32 * L - 1) > plan.P          # two's complement holds (-P, P)
            assert sum(info.P_limbs[t] << (32 * t) for t in range(L)) == plan.P
            for l, w in enumerate(plan.w):
                assert sum(info.w_limbs[l][t] << (32 * t) for t in range(L)) == w
        # fast mode's per-side budget H = RD64((P-1)/2) (R15)
        assert Fraction(info.fast_H) == scheme.fast_H(plan)


def test_karatsuba_scheme_plan(oz2mod):
    """OZ2_SCHEME_FP8_KARATSUBA: the planner's moduli, P and CRT weights equal
    the oracle's Karatsuba family; no squares, 3 digit planes per modulus."""
    from fractions import Fraction
    from oracle import moduli as mod
    assert oz2mod.oz2_set_scheme("karatsuba") == 0
    try:
        assert oz2mod.oz2_get_scheme() == oz2mod.OZ2_SCHEME_FP8_KARATSUBA
        for N in [2, 12, 13, 14, 20, 33]:
            assert oz2mod.oz2_moduli(N) == mod.karatsuba_moduli(N)
            info = oz2mod.oz2_plan_query(N, 16384)
            plan = mod.crt_plan(mod.karatsuba_moduli(N))
            assert info.num_squares == 0 and info.num_planes == 3 * N
            assert Fraction(info.p_prime) == mod.p_prime(plan.P)
            L = info.num_limbs
            assert sum(info.P_limbs[t] << (32 * t) for t in range(L)) == plan.P
            for l, w in enumerate(plan.w):
                assert sum(info.w_limbs[l][t] << (32 * t) for t in range(L)) == w
    finally:
        oz2mod.oz2_set_scheme("fp8")
    assert oz2mod.oz2_set_scheme(3) == -1 and oz2mod.oz2_get_scheme() == oz2mod.OZ2_SCHEME_FP8


def test_mode_switch(oz2mod):
    assert oz2mod.oz2_get_mode() == oz2mod.OZ2_MODE_ACCURATE
    assert oz2mod.oz2_set_mode("fast") == 0 and oz2mod.oz2_get_mode() == oz2mod.OZ2_MODE_FAST
    assert oz2mod.oz2_set_mode(7) == -1 and oz2mod.oz2_get_mode() == oz2mod.OZ2_MODE_FAST
    assert oz2mod.oz2_set_mode("accurate") == 0 and oz2mod.oz2_get_mode() == oz2mod.OZ2_MODE_ACCURATE


def test_argument_errors_before_device(oz2mod):
    # BLAS xerbla order; returned before any device work
    assert oz2mod.oz2_dgemm("X", "N", 1, 1, 1, 1.0, 0, 1, 0, 1, 0.0, 0, 1, 12) == -1
    assert oz2mod.oz2_dgemm("N", "Q", 1, 1, 1, 1.0, 0, 1, 0, 1, 0.0, 0, 1, 12) == -2
    assert oz2mod.oz2_dgemm("N", "N", -1, 1, 1, 1.0, 0, 1, 0, 1, 0.0, 0, 1, 12) == -3
    assert oz2mod.oz2_dgemm("N", "N", 4, 1, 1, 1.0, 0, 3, 0, 1, 0.0, 0, 4, 12) == -8
    assert oz2mod.oz2_dgemm("N", "N", 4, 1, 5, 1.0, 0, 4, 0, 4, 0.0, 0, 4, 12) == -10
    assert oz2mod.oz2_dgemm("N", "N", 4, 1, 1, 1.0, 0, 4, 0, 1, 0.0, 0, 3, 12) == -13
    assert oz2mod.oz2_dgemm("N", "N", 4, 1, 1, 1.0, 0, 4, 0, 1, 0.0, 0, 4, 1) == -14
    assert oz2mod.oz2_dgemm("N", "N", 0, 0, 0, 1.0, 0, 1, 0, 1, 0.0, 0, 1, 12) == 0   # quick return
    assert oz2mod.oz2_workspace_size("N", "N", 64, 64, 64, 14) > 0


def test_blocking_planner(oz2mod):
    """m/n blocking: full workspace -> unblocked; smaller -> blocks that fit,
    multiples of 256 (or the full extent), with the largest column block first."""
    for (m, n, k, N) in [(16384, 16384, 16384, 13), (5000, 3000, 777, 12), (300, 70000, 4096, 16)]:
        full = oz2mod.oz2_workspace_size("N", "N", m, n, k, N)
        assert oz2mod.oz2_workspace_size_blocked(m, n, k, N, 0, 0) == full
        assert oz2mod.oz2_plan_blocking(m, n, k, N, full) == (0, m, n)
        prev = None
        for frac in [0.9, 0.5, 0.25, 0.1, 0.03]:
            rc, mb, nb = oz2mod.oz2_plan_blocking(m, n, k, N, int(full * frac))
            if rc != 0:
                assert rc == oz2mod.OZ2_ERR_WORKSPACE
                assert oz2mod.oz2_workspace_size_blocked(m, n, k, N, 256, 256) > int(full * frac)
                continue
            assert (mb == m or mb % 256 == 0) and (nb == n or nb % 256 == 0)
            assert 0 < mb <= m and 0 < nb <= n and (mb, nb) != (m, n)
            assert oz2mod.oz2_workspace_size_blocked(m, n, k, N, mb, nb) <= int(full * frac)
            # maximal: one more 256-row slab of A would not fit (unless mb is already m)
            if mb < m:
                assert oz2mod.oz2_workspace_size_blocked(m, n, k, N, mb + 256, nb) > int(full * frac)
            if prev:
                assert mb * nb <= prev[0] * prev[1]
            prev = (mb, nb)
    # too small for anything
    assert oz2mod.oz2_plan_blocking(4096, 4096, 4096, 13, 1 << 20)[0] == oz2mod.OZ2_ERR_WORKSPACE
    assert oz2mod.oz2_set_blocking(100, 0) == -1 and oz2mod.oz2_set_blocking(0, 300) == -2
    assert oz2mod.oz2_set_blocking(0, 0) == 0


def test_int8_scheme_plan_matches_oracle(oz2mod):
    """INT8 scheme (NEXT-3): moduli, planes (one per modulus), P, CRT weights and fast_H
    of the host planner equal the oracle's; the scheme switch is per thread."""
    from fractions import Fraction
    from oracle import int8, moduli as mod, scheme
    assert oz2mod.oz2_get_scheme() == oz2mod.OZ2_SCHEME_FP8
    assert oz2mod.oz2_set_scheme(5) == -1
    assert oz2mod.oz2_set_scheme("int8") == 0
    try:
        for N in [2, 14, 15, 16, 20, 33]:
            assert oz2mod.oz2_moduli(N) == mod.int8_moduli(N)
            info = oz2mod.oz2_plan_query(N, 4096)
            pl = int8.plan(N)
            assert info.num_planes == N and info.num_squares == 0
            L = info.num_limbs
            assert sum(info.P_limbs[t] << (32 * t) for t in range(L)) == pl.P
            for l, w in enumerate(pl.w):
                assert sum(info.w_limbs[l][t] << (32 * t) for t in range(L)) == w
            assert Fraction(info.fast_H) == scheme.fast_H(pl)
        # workspace: N planes per operand instead of M_N
        w8 = oz2mod.oz2_workspace_size("N", "N", 4096, 4096, 4096, 14)
    finally:
        oz2mod.oz2_set_scheme("fp8")
    w_fp8 = oz2mod.oz2_workspace_size("N", "N", 4096, 4096, 4096, 14)
    assert w8 < w_fp8


def test_tuning_knobs_host_only(oz2mod):
    """oz2_set_tuning validates knob and range, oz2_get_tuning reads back, reset restores
    the defaults (include/oz2.h OZ2_TUNE_*); no environment variable is consulted."""
    P = oz2mod
    P.oz2_reset_tuning()
    defaults = {k: P.oz2_get_tuning(k) for k in P.TUNE}
    assert defaults["cta_group"] == 2 and defaults["mod_split"] == -1 and defaults["sq_order"] == 1
    assert P.oz2_set_tuning("cta_group", 3) == -2
    assert P.oz2_set_tuning(99, 1) == -1
    assert P.oz2_set_tuning("sync_chunk", 0) == -2
    assert P.oz2_set_tuning("tile_n", 384) == -2 and P.oz2_set_tuning("tile_n", 128) == -2
    assert len(P.TUNE) == 17 and P.TUNE["tile_n"] == 16
    assert P.oz2_set_tuning("cta_group", 1) == 0 and P.oz2_get_tuning("cta_group") == 1
    with P.tuning(mod_split=2, fused_crt=0):
        assert P.oz2_get_tuning("mod_split") == 2 and P.oz2_get_tuning("fused_crt") == 0
    assert P.oz2_get_tuning("mod_split") == -1
    P.oz2_reset_tuning()
    assert {k: P.oz2_get_tuning(k) for k in P.TUNE} == defaults
    src = open(os.path.join(ROOT, "paper_2603_10634_b200", "csrc", "oz2_api.cu")).read()
    for f in ["oz2_api.cu", "gemm_kernel.cu", "crt_kernel.cu", "prep_kernels.cu"]:
        src = open(os.path.join(ROOT, "paper_2603_10634_b200", "csrc", f)).read()
        assert "getenv" not in src, f


def test_options_struct_layout(oz2mod):
    """The ctypes mirror of oz2_options has the C layout: 13 pointers, timing_ms, four
    int32 settings and four reserved int32 (x86-64: 14 * 8 + 8 * 4 = 144 bytes)."""
    import ctypes
    assert ctypes.sizeof(oz2mod.oz2_options) == 14 * 8 + 8 * 4
