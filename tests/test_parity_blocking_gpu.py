"""m/n blocking (workspace reduction) through the C ABI.

Steps 1-3 always run on the whole problem, so a blocked call must give exactly the
unblocked call's exponents and C (bit for bit), and C must equal the oracle's."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import scheme
from synth import gen_device, gen_host

from gpu_helpers import run


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_10634_b200 as P
    P.lib()
    yield P
    P.oz2_set_blocking(0, 0)


def _run_blocked(P, A, B, N, mb, nb, **kw):
    P.oz2_set_blocking(mb, nb)
    try:
        out = run(A, B, N, want_residues=False, **kw)
        got = P.oz2_get_blocking()
    finally:
        P.oz2_set_blocking(0, 0)
    return out, got


@pytest.mark.parametrize("mode", ["accurate", "fast"])
@pytest.mark.parametrize("mb,nb", [(256, 512), (512, 256), (256, 0), (0, 256)])
def test_blocked_equals_oracle(dev, mode, mb, nb):
    m, k, n = 700, 300, 900
    A = gen_host(m, k, "phi", phi=1.0, seed=41, order="F")
    B = gen_host(k, n, "phi", phi=1.0, seed=42, order="F")
    ref = scheme.dgemm(A, B, 13, mode=mode)
    out, got = _run_blocked(dev, A, B, 13, mb, nb, mode=mode)
    assert got == (mb or m, nb or n)
    if mode == "fast":
        # fast-mode exponents are exact integer decisions: C equals the oracle's outright
        assert out["e_mu"].tolist() == ref.e_mu and out["e_nu"].tolist() == ref.e_nu
        assert np.array_equal(out["C"], ref.C)
    else:
        # accurate mode: import the oracle's exponents (R13) -> blocked steps 4-6 exact
        imp, _ = _run_blocked(dev, A, B, 13, mb, nb, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu)
        assert np.array_equal(imp["C"], ref.C)
    full = run(A, B, 13, mode=mode)
    assert np.array_equal(out["e_mu"], full["e_mu"]) and np.array_equal(out["e_nu"], full["e_nu"])
    assert np.array_equal(out["C"], full["C"])


@pytest.mark.parametrize("ta,tb", [("T", "N"), ("N", "T"), ("T", "T")])
def test_blocked_layouts_alpha_beta(dev, ta, tb):
    m, k, n = 600, 200, 530
    A = gen_host(m, k, "phi", phi=2.0, seed=43, order="F")
    B = gen_host(k, n, "phi", phi=2.0, seed=44, order="F")
    C0 = gen_host(m, n, "uniform", seed=45, order="F")
    kw = dict(transa=ta, transb=tb, alpha=0.5, beta=-2.0, C0=C0, ldc_pad=3)
    out, _ = _run_blocked(dev, A, B, 12, 256, 256, **kw)
    full = run(A, B, 12, **kw)
    assert np.array_equal(out["C"], full["C"])
    assert np.array_equal(out["C_pad"], full["C_pad"])       # rows beyond m untouched


def test_blocked_fused_crt_path(dev, knobs):
    """k >= 8192 with the fused CRT forced takes the CRT-in-epilogue path; blocks of 512 x 768."""
    knobs(fused_crt=1, mod_split=0)
    m, k, n = 1100, 8192, 1300
    A = gen_host(m, k, "phi", phi=0.5, seed=46, order="F")
    B = gen_host(k, n, "phi", phi=0.5, seed=47, order="F")
    out, got = _run_blocked(dev, A, B, 13, 512, 768)
    assert got == (512, 768)
    full = run(A, B, 13)
    assert np.array_equal(out["C"], full["C"])


def test_auto_blocking_from_small_workspace(dev):
    """A user workspace below oz2_workspace_size makes the call block itself."""
    import torch
    P = dev
    m = n = k = 4096
    N = 13
    A = gen_device(m, k, "phi", phi=1.0, seed=48)
    B = gen_device(k, n, "phi", phi=1.0, seed=49)
    C1 = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    C2 = torch.empty_like(C1)
    P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    full = P.oz2_workspace_size("N", "N", m, n, k, N)
    ws = torch.empty(full, dtype=torch.uint8, device="cuda")
    P.oz2_set_workspace(ws.data_ptr(), full)
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C1.data_ptr(), m, N) == 0
    assert P.oz2_get_blocking() == (m, n)
    small = full // 4
    rc, mb, nb = P.oz2_plan_blocking(m, n, k, N, small)
    assert rc == 0 and (mb, nb) != (m, n)
    P.oz2_set_workspace(ws.data_ptr(), small)
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C2.data_ptr(), m, N) == 0
    assert P.oz2_get_blocking() == (mb, nb)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    # too small for any blocking
    P.oz2_set_workspace(ws.data_ptr(), 1 << 20)
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C2.data_ptr(), m, N) \
        == P.OZ2_ERR_WORKSPACE
    P.oz2_set_workspace(None, 0)


def test_debug_outputs_force_unblocked(dev):
    A = gen_host(300, 100, "phi", phi=1.0, seed=50, order="F")
    B = gen_host(100, 280, "phi", phi=1.0, seed=51, order="F")
    dev.oz2_set_blocking(256, 256)
    try:
        out = run(A, B, 12)                 # asks for the whole-problem residues
        assert dev.oz2_get_blocking() == (300, 280)
    finally:
        dev.oz2_set_blocking(0, 0)
    from sampled import check_sampled
    check_sampled(A, B, 12, list(range(300)), list(range(280)),
                  {"e_mu": out["e_mu"], "e_nu": out["e_nu"], "C": out["C"],
                   "res": out["residues"]}, accuracy=False)


@pytest.mark.parametrize("sch", ["int8", "karatsuba"])
@pytest.mark.parametrize("mode", ["accurate", "fast"])
@pytest.mark.parametrize("mb,nb", [(256, 512), (512, 256)])
def test_blocked_other_schemes(dev, sch, mode, mb, nb):
    """The INT8 and Karatsuba-only schemes through m/n blocks: C and exponents identical to
    the unblocked call of the same scheme, and the oracle's on one sampled entry per tile."""
    m, k, n = 700, 900, 800
    A = gen_host(m, k, "phi", phi=1.0, seed=95)
    B = gen_host(k, n, "phi", phi=1.0, seed=96)
    out, got = _run_blocked(dev, A, B, 14, mb, nb, scheme=sch, mode=mode)
    assert got == (mb, nb)
    full = run(A, B, 14, scheme=sch, mode=mode)
    assert np.array_equal(out["e_mu"], full["e_mu"]) and np.array_equal(out["e_nu"], full["e_nu"])
    assert np.array_equal(out["C"], full["C"])
    from sampled import check_sampled, col_cover, tile_cover
    I, J = tile_cover(m), col_cover(n)
    check_sampled(A, B, 14, I, J, {"e_mu": out["e_mu"], "e_nu": out["e_nu"],
                                   "C": out["C"][np.ix_(I, J)]},
                  family="int8" if sch == "int8" else "karatsuba", mode=mode, accuracy=False)
