"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(oz2_dgemm on device buffers, default kernels), on sampled outputs the oracle computes
one by one: the exponents of the sampled rows/columns (each needs a full row of
A-bar B-bar), the residues C'_l and the final C of the sampled entries.  Residues and C
must be bit-exact wherever the exponents agree (reading R13); exponents must agree on
all but a vanishing fraction (the R6 rounding window).  Accuracy against the exact
product is checked against the closed-form a-priori bound."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import exact, scheme
from synth import gen_device
from sampled import check_sampled, col_cover, tile_cover


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_10634_b200 as P
    P.lib()
    return P


def _run_sampled(P, m, k, n, N, phi, seed, I, J, mode="accurate"):
    import torch
    A = gen_device(m, k, "phi", phi=phi, seed=seed)
    B = gen_device(k, n, "phi", phi=phi, seed=seed + 1)
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    e_mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    e_nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    res = torch.zeros(N * n * m, dtype=torch.int16, device="cuda")
    opt = P.oz2_options()
    opt.e_mu = e_mu.data_ptr()
    opt.e_nu = e_nu.data_ptr()
    opt.residues = res.data_ptr()
    P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    P.oz2_set_workspace(None, 0)
    assert P.oz2_set_mode(mode) == 0
    try:
        rc = P.oz2_dgemm_ex("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                            C.data_ptr(), m, N, opt)
    finally:
        P.oz2_set_mode("accurate")
    assert rc == 0
    torch.cuda.synchronize()
    It = torch.tensor(I, device="cuda")
    Jt = torch.tensor(J, device="cuda")
    res3 = res.view(N, n, m)
    out = {
        "C": C[It][:, Jt].cpu().numpy(),
        "e_mu": e_mu.cpu().numpy(),
        "e_nu": e_nu.cpu().numpy(),
        "res": res3[:, Jt][:, :, It].permute(0, 2, 1).cpu().numpy(),     # [l][a][b]
        "A_rows": A[It].cpu().numpy(),
        "B_cols": B[:, Jt].cpu().numpy(),
        "A": A.cpu().numpy(),
        "B": B.cpu().numpy(),
    }
    del A, B, C, res, res3
    torch.cuda.empty_cache()
    P.oz2_finalize()
    return out


def _fast_exps(X, rows, N):
    """Oracle fast-mode exponents of the selected rows of X (R15: each is row-local)."""
    plan, _, _ = scheme.plan_constants(N)
    Xs = X[rows]
    e_prime, codes = scheme.prescale_rows(Xs)
    zero = [not np.any(r) for r in Xs]
    return scheme.fast_exponents(e_prime, codes, plan, zero)


def _check(out, N, I, J, mode="accurate"):
    return check_sampled(out["A"], out["B"], N, I, J, out, mode=mode)


@pytest.mark.parametrize("phi", [0.0, 4.0])
def test_config2_8192_moduli_sweep(dev, phi):
    """BASELINE config 2: m=n=k=8192, N in 12..20, accuracy vs exact falls with N.  At
    N = 13 the sample covers every 256 x 256 tile (the hybrid schedule: 13 full waves
    tile-major, the ragged last wave split into (tile, modulus) items, separate CRT)."""
    m = n = k = 8192
    errs = []
    for N in [12, 13, 16, 20]:
        if N == 13:
            I, J = tile_cover(m), col_cover(n)
        else:
            I, J = [0, 4097, 8191], [1, 5000, 8190]
        out = _run_sampled(dev, m, k, n, N, phi, 11, I, J)
        e = _check(out, N, I, J)
        if N != 13:
            errs.append(e)
    assert errs[1] <= errs[0] and errs[2] <= max(errs[1], 2e-17)


def test_config3_16384_bench_workload(dev):
    """BASELINE config 3 as bench.py runs it (m=n=k=16384, phi=1, N=13, default kernels:
    CTA pairs, tile-major persistent schedule with the CRT fused and deferred into the
    next tile's epilogues): 64 x 64 sampled entries, one per output tile -- every tile,
    both CTAs of each pair, all four TMEM lane quadrants, both epilogue column halves."""
    I, J = tile_cover(16384), col_cover(16384)
    assert len(I) == len(J) == 64
    out = _run_sampled(dev, 16384, 16384, 16384, 13, 1.0, 21, I, J)
    err = _check(out, 13, I, J)
    assert err < 1e-15


@pytest.mark.parametrize("N,phi", [(12, 0.0), (13, 1.0)])
def test_config4_large_k_65536(dev, N, phi):
    """BASELINE config 4: m=n=4096, k=65536 -- the FP32 exactness limit k = 2^16; every
    tile sampled."""
    I, J = tile_cover(4096), col_cover(4096)
    out = _run_sampled(dev, 4096, 65536, 4096, N, phi, 31, I, J)
    _check(out, N, I, J)


@pytest.mark.parametrize("N", [13, 16])
def test_config3_16384_fast_mode(dev, N):
    """Fast mode (R15) at the bench workload: exponents, residues and C bit-exact on the
    sampled entries; fast mode with N = 13 stays within the FP64-level band."""
    I, J = tile_cover(16384)[::4], col_cover(16384)[1::4]
    out = _run_sampled(dev, 16384, 16384, 16384, N, 1.0, 21, I, J, mode="fast")
    err = _check(out, N, I, J, mode="fast")
    assert err < 1e-14


def test_config4_large_k_65536_fast_mode(dev):
    I, J = [0, 2048, 4095], [7, 4000]
    out = _run_sampled(dev, 4096, 65536, 4096, 13, 4.0, 31, I, J, mode="fast")
    _check(out, 13, I, J, mode="fast")


def _run_fast_light(P, m, k, n, N, phi, seed, I, J, rows=None):
    """Fast mode without debug outputs (the bench's launch configuration, whatever blocking
    the library picks); returns the sampled rows/columns of A, B and C.  rows = (r0, r1)
    runs only that row block of A (a rank's shard of the row-sharded driver)."""
    import torch
    A = gen_device(m, k, "phi", phi=phi, seed=seed)
    B = gen_device(k, n, "phi", phi=phi, seed=seed + 1)
    r0, r1 = rows if rows else (0, m)
    mm = r1 - r0
    C = torch.empty((n, mm), dtype=torch.float64, device="cuda").t()
    P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    P.oz2_set_workspace(None, 0)
    assert P.oz2_set_mode("fast") == 0
    try:
        rc = P.oz2_dgemm("N", "N", mm, n, k, 1.0, A[r0:].data_ptr(), m, B.data_ptr(), k, 0.0,
                         C.data_ptr(), mm, N)
    finally:
        P.oz2_set_mode("accurate")
    assert rc == 0
    torch.cuda.synchronize()
    It = torch.tensor([i - r0 for i in I], device="cuda")
    Jt = torch.tensor(J, device="cuda")
    out = {"C": C[It][:, Jt].cpu().numpy(), "A_rows": A[torch.tensor(I, device="cuda")].cpu().numpy(),
           "B_cols": B[:, Jt].cpu().numpy()}
    del A, B, C
    torch.cuda.empty_cache()
    P.oz2_finalize()
    return out


def _check_light(out, N, nI, nJ):
    Ar, Bc = out["A_rows"], out["B_cols"]
    emu, enu = _fast_exps(Ar, list(range(nI)), N), _fast_exps(Bc.T.copy(), list(range(nJ)), N)
    _, Cref = scheme.entries(Ar, Bc, N, list(range(nI)), list(range(nJ)), list(emu), list(enu))
    assert np.array_equal(out["C"], Cref)
    ex = exact.exact_entries(Ar, Bc, range(nI), range(nJ))
    bound = exact.apriori_bound(Ar, Bc, list(emu), list(enu))
    assert np.all(np.abs(out["C"] - ex) <= 2 * bound + np.abs(ex) * 2.0 ** -52)
    return float(np.linalg.norm(out["C"] - ex) / np.linalg.norm(ex))


def test_config5_32768_fast_sampled(dev):
    """BASELINE config 5's problem (m=n=k=32768, N=13) on one B200 in fast mode (both
    scaling vectors row/column-local, R15): sampled C bit-exact against the oracle."""
    I, J = [0, 20000, 32767], [5, 32760]
    out = _run_fast_light(dev, 32768, 32768, 32768, 13, 1.0, 41, I, J)
    assert _check_light(out, 13, len(I), len(J)) < 1e-15


def test_config5_rank_shard_fast_equals_unsharded(dev):
    """One rank's shard of the row-sharded driver (rows [8192, 16384) of a G=4 split): in
    fast mode mu and nu are row/column-local, so the shard's C equals the same rows of
    the unsharded call bit for bit (in accurate mode nu is block-local instead, R13)."""
    m = n = k = 8192 * 2
    I, J = [8192, 12000, 16383], [3, 16000]
    shard = _run_fast_light(dev, m * 2, k, n, 13, 1.0, 43, I, J, rows=(8192, 16384))
    full = _run_fast_light(dev, m * 2, k, n, 13, 1.0, 43, I, J)
    assert np.array_equal(shard["C"], full["C"])
    _check_light(full, 13, len(I), len(J))


def test_karatsuba_16384_fast_sampled(dev):
    """The Karatsuba-only family at the bench size in fast mode (exponents decided in exact
    integers, R15): sampled C bit-exact against oracle.scheme with family="karatsuba"."""
    N = 13
    I, J = [7, 9001, 16383], [2, 15000]
    dev.oz2_set_scheme("karatsuba")
    try:
        out = _run_fast_light(dev, 16384, 16384, 16384, N, 1.0, 51, I, J)
    finally:
        dev.oz2_set_scheme("fp8")
    Ar, Bc = out["A_rows"], out["B_cols"]
    plan, _, _ = scheme.plan_constants(N, "karatsuba")
    eA, cA = scheme.prescale_rows(Ar)
    eB, cB = scheme.prescale_rows(Bc.T.copy())
    emu = scheme.fast_exponents(eA, cA, plan, [False] * len(I))
    enu = scheme.fast_exponents(eB, cB, plan, [False] * len(J))
    _, Cref = scheme.entries(Ar, Bc, N, list(range(len(I))), list(range(len(J))), emu, enu, family="karatsuba")
    assert np.array_equal(out["C"], Cref)
    ex = exact.exact_entries(Ar, Bc, range(len(I)), range(len(J)))
    assert np.linalg.norm(out["C"] - ex) / np.linalg.norm(ex) < 2e-15


def test_int8_config4_fast_sampled(dev):
    """The INT8 scheme at config 4's shape (m = n = 4096, k = 65536 = its exactness limit),
    fast mode: sampled C bit-exact against oracle.int8's definition (exponents from the
    integer sums of squares of the U8 bounds, R16)."""
    from oracle import int8
    N = 15
    I, J = [0, 2049, 4095], [5, 3000]
    dev.oz2_set_scheme("int8")
    try:
        out = _run_fast_light(dev, 4096, 65536, 4096, N, 1.0, 53, I, J)
    finally:
        dev.oz2_set_scheme("fp8")
    Ar, Bc = out["A_rows"], out["B_cols"]
    pl = int8.plan(N)
    eA, bA = int8.prescale_rows(Ar)
    eB, bB = int8.prescale_rows(Bc.T.copy())
    emu = int8.exponents(eA, [int(sum(int(v) ** 2 for v in r)) for r in bA], pl, [False] * len(I))
    enu = int8.exponents(eB, [int(sum(int(v) ** 2 for v in r)) for r in bB], pl, [False] * len(J))
    Aint = scheme.to_integral(Ar, emu)
    BintT = scheme.to_integral(Bc.T.copy(), enu)
    res = [scheme.modprod_direct(scheme.residues(Aint, p), scheme.residues(BintT, p), p) for p in pl.moduli]
    Cref = scheme.inverse_scale(scheme.crt_combine(res, pl), emu, enu)
    assert np.array_equal(out["C"], Cref)
