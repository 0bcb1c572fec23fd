"""Step 1 (prescale, eq. def:mu'nu') through the C ABI: the one-read form
(chunk-local casts + rescale to the row exponent, OZ2_TUNE_PRESCALE_2READ = 0) against the
oracle and against the two-read form (row maxima, then the cast; the default), on
rows whose entries span the whole binary64 range -- so chunk exponents differ from the row
exponent by 0 .. > 1000, rescaled codes land on every part of the E4M3 grid (normal,
subnormal, the 2^-9 floor) -- with zero chunks, zero rows, NaN / Inf rows, both storage
orders, k across the 2048-byte super-chunk boundary, and both FP8 and INT8 schemes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import int8 as oint8
from oracle import scheme
from synth import gen_host


def _wide(rows, k, seed):
    """Entries (rand - 0.5) 2^t with t uniform in [-60, 60] per element, plus rows with
    single huge / subnormal outliers and zero stretches longer than a 128-wide chunk."""
    rng = np.random.default_rng(seed)
    X = gen_host(rows, k, "uniform", seed=seed) * np.exp2(rng.integers(-60, 61, size=(rows, k)))
    X[1, :] = 0.0                                   # zero row (R3)
    X[2, 300:700] = 0.0                             # zero chunks inside a nonzero row
    X[3, 5] = 2.0 ** 1000                           # one huge entry: every other chunk rescales by ~1000
    X[4, :] *= 2.0 ** -1000                         # near the subnormal range ...
    X[4, 7] = 2.0 ** -1070                          # ... and a subnormal
    X[5, :] = 0.0
    X[5, k - 1] = -3.0                              # a single nonzero, in the ragged last chunk
    X[6, ::2] *= 2.0 ** -40                         # alternating magnitudes within each chunk
    return X


def _run(A, B, N, two_read, transa="N", transb="N", scheme_name="fp8"):
    import paper_2603_10634_b200 as P
    from gpu_helpers import run
    assert P.oz2_set_tuning("prescale_2read", 1 if two_read else 0) == 0
    try:
        return run(A, B, N, transa=transa, transb=transb, want_residues=False, scheme=scheme_name)
    finally:
        P.oz2_reset_tuning()


@pytest.mark.parametrize("transa,transb", [("N", "N"), ("T", "T")])
@pytest.mark.parametrize("k", [2300, 700])
def test_one_read_prescale_matches_oracle(transa, transb, k):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n = 130, 70
    A = _wide(m, k, 5)
    B = _wide(n, k, 6).T.copy()
    res = _run(A, B, 13, False, transa, transb)
    epa, abar = scheme.prescale_rows(A)
    epb, bbar = scheme.prescale_rows(B.T)
    assert res["e_prime_a"].tolist() == epa and res["e_prime_b"].tolist() == epb
    assert np.array_equal(res["abar"], abar) and np.array_equal(res["bbar"], bbar)
    two = _run(A, B, 13, True, transa, transb)
    for key in ("abar", "bbar", "e_prime_a", "e_prime_b", "rmax", "smax", "e_mu", "e_nu", "C"):
        assert np.array_equal(res[key], two[key]), key


def test_one_read_prescale_int8_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n, k = 96, 64, 2300
    A = _wide(m, k, 7)
    B = _wide(n, k, 8).T.copy()
    res = _run(A, B, 15, False, scheme_name="int8")
    epa, abar = oint8.prescale_rows(A)
    epb, bbar = oint8.prescale_rows(B.T)
    assert res["e_prime_a"].tolist() == epa and res["e_prime_b"].tolist() == epb
    assert np.array_equal(res["abar"].astype(np.int64), abar)
    assert np.array_equal(res["bbar"].astype(np.int64), bbar)
    two = _run(A, B, 15, True, scheme_name="int8")
    for key in ("abar", "bbar", "e_mu", "e_nu", "C"):
        assert np.array_equal(res[key], two[key]), key


@pytest.mark.parametrize("sch", ["fp8", "int8"])
def test_one_read_prescale_nonfinite(sch):
    """NaN / Inf rows and columns (R12): the same A-bar (zero bounds on those rows), status
    and C as the two-read form."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n, k = 70, 50, 2300
    A = _wide(m, k, 9)
    B = _wide(n, k, 10).T.copy()
    A[8, 2000] = np.nan
    A[9, 3] = np.inf
    B[100, 4] = -np.inf
    N = 15 if sch == "int8" else 13
    one = _run(A, B, N, False, scheme_name=sch)
    two = _run(A, B, N, True, scheme_name=sch)
    assert one["status"] != 0 and two["status"] != 0
    for key in ("abar", "bbar", "e_prime_a", "e_prime_b", "e_mu", "e_nu"):
        assert np.array_equal(one[key], two[key]), key
    assert np.all(one["abar"][8] == 0) and np.all(one["abar"][9] == 0)
    assert np.array_equal(np.isnan(one["C"]), np.isnan(two["C"]))
    fin = ~np.isnan(two["C"])
    assert np.array_equal(one["C"][fin], two["C"][fin])


@pytest.mark.parametrize("sch,N", [("fp8", 13), ("int8", 15), ("karatsuba", 13)])
def test_digits_fma_fast_path_identical(sch, N):
    """Step 4's one-FMA scale-and-truncate path (OZ2_TUNE_DIGITS_FMA = 1, chosen per row from
    step 1's row maximum) gives the same digit planes, residues and C as the general path,
    on rows that take either path (wide exponent spread, huge / subnormal outliers)."""
    import torch
    import paper_2603_10634_b200 as P
    from gpu_helpers import run
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n, k = 100, 90, 2300
    A = _wide(m, k, 11)
    B = _wide(n, k, 12).T.copy()
    outs = []
    for v in (0, 1):
        assert P.oz2_set_tuning("digits_fma", v) == 0
        try:
            outs.append(run(A, B, N, want_digits=True, scheme=sch))
        finally:
            P.oz2_reset_tuning()
    for key in ("digits_a", "digits_b", "residues", "e_mu", "e_nu", "C"):
        assert np.array_equal(outs[0][key], outs[1][key]), key


def test_digits_fma_fast_path_blocked():
    """The fast path reads step 1's row maxima in step 4; with m/n blocking (several row and
    column blocks, so A's digits are recomputed after earlier blocks' GEMMs have run) C must
    equal the unblocked general-path result bit for bit."""
    import torch
    import paper_2603_10634_b200 as P
    from gpu_helpers import run
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n, k = 600, 520, 2300
    A = _wide(m, k, 13)
    B = _wide(n, k, 14).T.copy()
    ref = run(A, B, 13, want_residues=False)
    assert P.oz2_set_tuning("digits_fma", 1) == 0 and P.oz2_set_blocking(256, 256) == 0
    try:
        blk = run(A, B, 13, want_residues=False)
    finally:
        P.oz2_reset_tuning()
        P.oz2_set_blocking(0, 0)
    assert np.array_equal(ref["C"], blk["C"])


@pytest.mark.parametrize("transa,transb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("k", [701, 2300])
@pytest.mark.parametrize("sch", ["fp8", "int8"])
def test_two_read_cast_matches_oracle(transa, transb, k, sch):
    """The default step 1 (k_rowmax, then k_cast: a lane casts 16 consecutive k of a row with
    the integer E4M3 round-up; zeros, sub-2^-6 results and subnormal inputs on the slow path)
    against the oracle's prescale: e' and A-bar / B-bar bit-exact for both storage orders of
    both operands, k odd (K-major operands then have an odd leading dimension: scalar loads)
    and even (16-byte loads), wide exponent spread with zero / huge / subnormal outliers."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m, n = 97, 70
    A = _wide(m, k, 15)
    B = _wide(n, k, 16).T.copy()
    res = _run(A, B, 13 if sch == "fp8" else 15, True, transa, transb, scheme_name=sch)
    pre = scheme.prescale_rows if sch == "fp8" else oint8.prescale_rows
    epa, abar = pre(A)
    epb, bbar = pre(B.T)
    assert res["e_prime_a"].tolist() == list(epa) and res["e_prime_b"].tolist() == list(epb)
    assert np.array_equal(res["abar"].astype(np.int64), np.asarray(abar).astype(np.int64))
    assert np.array_equal(res["bbar"].astype(np.int64), np.asarray(bbar).astype(np.int64))
