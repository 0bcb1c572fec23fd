"""GPU parity of the FP8 scheme with the Karatsuba-only moduli (eq.
p_list_karatsuba P:264-276: 513, 512, 511, ...; every modulus takes the 3-digit Karatsuba
split with s = 16 and eq. C'-Karatsuba) through the C ABI, against
oracle.scheme.dgemm(family="karatsuba").  Same bars as the hybrid family
(tests/test_parity_gpu.py): prescale, digit planes, residues and C bit-exact; exponents
equal up to the R13 fallback; imported exponents bit-exact everywhere."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import moduli as mod, scheme
from synth import gen_host

from gpu_helpers import run
from test_parity_gpu import _codes_e4m3, _compare


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_10634_b200 as P
    P.lib()
    yield P
    P.oz2_set_scheme("fp8")


@pytest.mark.parametrize("seed", [0, 1])
def test_karatsuba_64cubed_N14_digits(dev, seed):
    """Config-1 shape with the Karatsuba family: every digit plane (3 per modulus,
    including p = 513 with |r| = 256 and the even p = 512), residues and C bit-exact."""
    A = gen_host(64, 64, "uniform", seed=seed)
    B = gen_host(64, 64, "uniform", seed=100 + seed)
    ref = scheme.dgemm(A, B, 14, want_digits=True, family="karatsuba")
    res = run(A, B, 14, want_digits=True, scheme="karatsuba")
    assert _compare(res, ref, A, B, 14).all()
    planes_a = [pl for (da, db) in ref.extra["digits"] for pl in da]
    planes_b = [pl for (da, db) in ref.extra["digits"] for pl in db]
    assert len(planes_a) == 3 * 14
    for x, pl in enumerate(planes_a):
        assert np.array_equal(res["digits_a"][x], _codes_e4m3(pl)), x
    for x, pl in enumerate(planes_b):
        assert np.array_equal(res["digits_b"][x], _codes_e4m3(pl)), x


@pytest.mark.parametrize("transa,transb", [("N", "N"), ("T", "T")])
@pytest.mark.parametrize("N,phi,mode", [(13, 1.0, "accurate"), (14, 4.0, "accurate"), (13, 0.5, "fast")])
def test_karatsuba_ragged(dev, transa, transb, N, phi, mode):
    """Several tiles and ragged tails in m, n, k; both scaling modes."""
    m, k, n = 200, 300, 290
    A = gen_host(m, k, "phi", phi=phi, seed=13, order="C")
    B = gen_host(k, n, "phi", phi=phi, seed=14, order="C")
    ref = scheme.dgemm(A, B, N, family="karatsuba", mode=mode)
    res = run(A, B, N, transa, transb, scheme="karatsuba", mode=mode)
    if mode == "fast":
        # fast mode decides exponents in exact integers (R15): everything bit-exact
        assert res["e_mu"].tolist() == ref.e_mu and res["e_nu"].tolist() == ref.e_nu
        for l in range(N):
            assert np.array_equal(res["residues"][l], ref.residues[l]), l
        assert np.array_equal(res["C"], ref.C)
    else:
        assert _compare(res, ref, A, B, N).mean() > 0.98
    rel = np.linalg.norm(res["C"] - ref.C) / np.linalg.norm(ref.C)
    assert rel <= 1e-15


@pytest.mark.parametrize("N", [2, 7, 13, 20, 33])
def test_karatsuba_imported_exponents_bit_exact(dev, N):
    """Oracle exponents fed to the GPU: every residue and every element of C bit-exact."""
    m, k, n = 130, 257, 260
    A = gen_host(m, k, "phi", phi=2.0, seed=15)
    B = gen_host(k, n, "phi", phi=2.0, seed=16)
    ref = scheme.dgemm(A, B, N, family="karatsuba")
    res = run(A, B, N, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu, scheme="karatsuba")
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref.residues[l]), l
    assert np.array_equal(res["C"], ref.C)


def test_karatsuba_residue_extremes(dev):
    """Imported zero exponents (A' = A): integer inputs whose residues hit +-256 mod 513
    and the even modulus 512's asymmetric range ends; products checked against
    mod(A'B', p) from the definition."""
    N = 13
    ps = mod.karatsuba_moduli(N)
    rng = np.random.default_rng(5)
    m, k, n = 70, 130, 66
    A = rng.integers(-2 ** 40, 2 ** 40, size=(m, k)).astype(np.float64)
    B = rng.integers(-2 ** 40, 2 ** 40, size=(k, n)).astype(np.float64)
    A[0, :8] = [256, -256, 513 * 7 + 256, -(513 * 7 + 256), 256, -256, 255, -257]   # mod 513 / 512 edges
    B[:8, 0] = [256, -256, 256 + 512 * 3, -256 - 512 * 5, 255, -255, 1, -1]
    res = run(A, B, N, e_mu_in=[0] * m, e_nu_in=[0] * n, scheme="karatsuba")
    Aint = scheme.to_integral(A, [0] * m)
    BintT = scheme.to_integral(B.T.copy(), [0] * n)
    for l, p in enumerate(ps):
        want = scheme.modprod_direct(scheme.residues(Aint, p), scheme.residues(BintT, p), p)
        assert np.array_equal(res["residues"][l], want), p
