"""CPU checks of the sampled-parity machinery (tests/sampled.py) and of the vectorised
oracle twins it uses (scheme.to_integral_fast, residues_fast, the batched
row_exponents): each equals the plain definition, and check_sampled accepts the full
oracle's own output and rejects perturbed exponents, residues or C."""
import numpy as np
import pytest

from oracle import scheme
from sampled import check_sampled, col_cover, tile_cover
from synth import gen_host


def test_to_integral_and_residues_fast_equal_plain():
    for phi, scale in [(1.0, 0), (4.0, 0), (1.0, -1030), (2.0, 600)]:
        X = gen_host(7, 300, "phi", phi=phi, seed=3, order="C") * 2.0 ** scale
        X[2, 5] = 0.0
        X[3, :] = 5e-324 * (X[3, :] > 0)           # subnormals
        exps = [40, 55, -3, 1074 + 40, 0, 60, 10]
        if scale > 0:
            exps = [e - 600 for e in exps]
        fast = scheme.to_integral_fast(X, exps)
        plain = scheme.to_integral(X, exps)
        if fast is None:
            continue
        assert np.array_equal(fast.astype(object), plain)
        for p in [1089, 1024, 961, 511, 256, 255, 2]:
            assert np.array_equal(scheme.residues_fast(fast, p), scheme.residues(plain, p))
    # out of int64 range -> None (callers fall back to Python ints)
    assert scheme.to_integral_fast(np.array([[1.0]]), [70]) is None


def test_row_exponents_batched_equals_full_oracle():
    A = gen_host(40, 200, "phi", phi=2.0, seed=5, order="C")
    B = gen_host(200, 30, "phi", phi=2.0, seed=6, order="C")
    A[4, :] = 0.0
    r = scheme.dgemm(A, B, 13)
    eA, emu, _ = scheme.row_exponents(A, range(40), B.T.copy(), 13)
    eB, enu, _ = scheme.row_exponents(B.T.copy(), range(30), A, 13)
    assert eA == r.e_prime_A and emu == r.e_mu and eB == r.e_prime_B and enu == r.e_nu


def test_tile_cover_hits_every_tile_half_and_quadrant():
    I = tile_cover(16384)
    J = col_cover(16384)
    assert [i // 256 for i in I] == list(range(64)) and [j // 256 for j in J] == list(range(64))
    assert {(i % 256) // 128 for i in I} == {0, 1}
    assert {((i % 128) // 32) for i in I} == {0, 1, 2, 3}
    assert {(j % 256) // 128 for j in J} == {0, 1}
    for ext in [1000, 300, 257, 5]:
        I = tile_cover(ext)
        assert all(0 <= i < ext for i in I) and len(I) == (ext + 255) // 256


def _fake_gpu(r, I, J):
    return {"e_mu": np.array(r.e_mu), "e_nu": np.array(r.e_nu),
            "res": np.array([R[np.ix_(I, J)] for R in r.residues]),
            "C": r.C[np.ix_(I, J)]}


def test_check_sampled_accepts_oracle_rejects_perturbations():
    m, k, n, N = 300, 257, 290, 13
    A = gen_host(m, k, "phi", phi=1.0, seed=7)
    B = gen_host(k, n, "phi", phi=1.0, seed=8)
    r = scheme.dgemm(A, B, N)
    I, J = tile_cover(m), col_cover(n)
    err = check_sampled(A, B, N, I, J, _fake_gpu(r, I, J))
    assert err < 1e-15
    g = _fake_gpu(r, I, J)
    g["C"] = g["C"].copy()
    g["C"][0, 1] = np.nextafter(g["C"][0, 1], np.inf)
    with pytest.raises(AssertionError):
        check_sampled(A, B, N, I, J, g)
    g = _fake_gpu(r, I, J)
    g["res"][3, 1, 0] += 1
    with pytest.raises(AssertionError):
        check_sampled(A, B, N, I, J, g)
    g = _fake_gpu(r, I, J)
    g["e_mu"] = g["e_mu"].copy()
    g["e_mu"][I[0]] += 1                        # outside the R6 window
    with pytest.raises(AssertionError):
        check_sampled(A, B, N, I, J, g)


def test_certify_rows_decides_the_condition():
    """The certification used for an exponent inside the R6 window: one below the
    oracle's exponent is certified (more headroom), two above is not."""
    from sampled import _certify_rows
    m, k, n, N = 20, 100, 24, 13
    A = gen_host(m, k, "phi", phi=1.0, seed=9)
    B = gen_host(k, n, "phi", phi=1.0, seed=10)
    r = scheme.dgemm(A, B, N)
    plan, _, _ = scheme.plan_constants(N)
    _certify_rows(A, [3], [r.e_mu[3] - 1], B.T.copy(), r.e_nu, plan.P)
    with pytest.raises(AssertionError):
        _certify_rows(A, [3], [r.e_mu[3] + 2], B.T.copy(), r.e_nu, plan.P)


@pytest.mark.parametrize("mode", ["accurate", "fast"])
def test_int8_sampled_path_equals_full_oracle(mode):
    from oracle import int8
    m, k, n, N = 270, 140, 300, 15
    A = gen_host(m, k, "phi", phi=2.0, seed=11)
    B = gen_host(k, n, "phi", phi=2.0, seed=12)
    A[7, :] = 0.0
    X = gen_host(5, 90, "phi", phi=4.0, seed=13, order="C")
    X[1, 3] = 5e-324
    e1, b1 = int8.prescale_rows(X)
    e2, b2 = int8.prescale_rows_fast(X)
    assert e1 == e2 and np.array_equal(b1, b2)
    r = int8.dgemm(A, B, N, mode=mode)
    I, J = tile_cover(m), col_cover(n)
    check_sampled(A, B, N, I, J, _fake_gpu(r, I, J), family="int8", mode=mode)
