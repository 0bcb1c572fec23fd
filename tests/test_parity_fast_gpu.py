"""GPU parity of fast mode (reading R15: Cauchy-Schwarz over the FP8 upper bounds, no
bound GEMM; Table 2's 3N-GEMM variant) through the C ABI.

Fast-mode exponents are decided in exact integer arithmetic on both sides (S_i is a sum
of E4M3 squares), so e_mu, e_nu must equal the oracle's everywhere, and with them the
residues and C are bit-exact (no R13 fallback needed)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import exact, scheme
from synth import gen_host

from gpu_helpers import run


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_10634_b200 as P
    P.lib()
    return P


def _check_fast(A, B, N, transa="N", transb="N", alpha=1.0, beta=0.0, C0=None):
    out = run(A, B, N, transa=transa, transb=transb, alpha=alpha, beta=beta, C0=C0, mode="fast")
    ref = scheme.dgemm(A, B, N, alpha=alpha, beta=beta, C=C0, mode="fast")
    assert out["e_prime_a"].tolist() == ref.e_prime_A
    assert out["e_prime_b"].tolist() == ref.e_prime_B
    assert out["e_mu"].tolist() == ref.e_mu
    assert out["e_nu"].tolist() == ref.e_nu
    for l in range(N):
        assert np.array_equal(out["residues"][l], ref.residues[l]), l
    assert np.array_equal(out["C"], ref.C)
    return out, ref


@pytest.mark.parametrize("m,k,n", [(64, 64, 64), (200, 300, 260), (513, 129, 37)])
@pytest.mark.parametrize("phi", [0.5, 4.0])
def test_fast_bit_exact(dev, m, k, n, phi):
    A = gen_host(m, k, "phi", phi=phi, seed=m + k, order="F")
    B = gen_host(k, n, "phi", phi=phi, seed=n + 7, order="F")
    _check_fast(A, B, 13)


@pytest.mark.parametrize("N", [2, 6, 12, 16, 20, 33])
def test_fast_moduli_range(dev, N):
    """Small and large P: H exact (N = 2) and truncated, t negative and positive."""
    A = gen_host(40, 150, "phi", phi=1.0, seed=N, order="F")
    B = gen_host(150, 30, "phi", phi=1.0, seed=N + 100, order="F")
    _check_fast(A, B, N)


@pytest.mark.parametrize("ta,tb", [("N", "T"), ("T", "N"), ("T", "T")])
def test_fast_layouts_alpha_beta(dev, ta, tb):
    A = gen_host(70, 90, "phi", phi=2.0, seed=5, order="F")
    B = gen_host(90, 50, "phi", phi=2.0, seed=6, order="F")
    C0 = gen_host(70, 50, "uniform", seed=7, order="F")
    _check_fast(A, B, 12, transa=ta, transb=tb, alpha=-0.75, beta=1.5, C0=C0)


def test_fast_zero_rows_and_tiny(dev):
    A = gen_host(48, 100, "phi", phi=1.0, seed=8, order="F")
    B = gen_host(100, 40, "phi", phi=1.0, seed=9, order="F")
    A[3, :] = 0.0
    B[:, 5] = 0.0
    A[7, :] *= 1e-300            # subnormal-range row: codes round up to 2^-9
    B[:, 9] *= 1e250
    out, ref = _check_fast(A, B, 13)
    assert out["e_mu"][3] == 0 and out["e_nu"][5] == 0


def test_fast_large_k_sum_of_squares(dev):
    """k = 65536 with every |a| at the top of its binade: S_i = k * 256^2 = 2^32 units of
    2^16, the largest sums the integer accumulator sees at the exactness limit."""
    m, k, n = 16, 65536, 24
    A = gen_host(m, k, "phi", phi=0.0, seed=10, order="F")
    B = gen_host(k, n, "phi", phi=0.0, seed=11, order="F")
    A[0, :] = 1.99
    B[:, 0] = -1.99
    out = run(A, B, 12, mode="fast")
    emu = scheme.fast_exponents(*scheme.prescale_rows(A), scheme.plan_constants(12)[0],
                                [False] * m)
    enu = scheme.fast_exponents(*scheme.prescale_rows(B.T.copy()), scheme.plan_constants(12)[0],
                                [False] * n)
    assert out["e_mu"].tolist() == emu and out["e_nu"].tolist() == enu
    I, J = [0, 5, 15], [0, 11, 23]
    _, Cref = scheme.entries(A, B, 12, I, J, [emu[i] for i in I], [enu[j] for j in J])
    assert np.array_equal(out["C"][np.ix_(I, J)], Cref)


def test_fast_vs_accurate_accuracy(dev):
    """fast mode over-estimates the bound, so at equal N it is no more accurate
    than accurate mode; it skips the bound GEMM (3N instead of 3N+1 FP8 GEMMs)."""
    A = gen_host(256, 2048, "phi", phi=2.0, seed=12, order="F")
    B = gen_host(2048, 256, "phi", phi=2.0, seed=13, order="F")
    I = list(range(0, 256, 17))
    J = list(range(0, 256, 19))
    ex = exact.exact_entries(A, B, I, J)
    errs = {}
    for mode in ["accurate", "fast"]:
        out = run(A, B, 12, mode=mode)
        C = out["C"][np.ix_(I, J)]
        errs[mode] = np.linalg.norm(C - ex) / np.linalg.norm(ex)
    assert errs["accurate"] <= errs["fast"]
