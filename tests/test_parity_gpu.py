"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bars:
  * e', A-bar, B-bar, digit planes, residues C'_l: bit-exact (integer/byte work);
  * R, S: sound (f_k R >= exact max) and within the R5 rounding budget;
  * e_mu, e_nu: equal to the oracle's (both take the FP32 round-down decisions of
    P:379-380); any row where the tensor core's FP32 rounding of C-bar' moves the
    floor is validated instead (several exponents are correct, reading R13);
  * C: bit-exact to the oracle wherever the exponents agree (the CRT is exact and the
    final rounding is RNE on both sides), hence normwise <= 1e-15 (north_star).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import exact, fp8, fp32, moduli as mod, scheme
from synth import gen_host


@pytest.fixture(scope="module", params=["cg1", "cg2", "cg4"])
def dev(request):
    """The library with each GEMM variant (OZ2_TUNE_CTA_GROUP, read per call): 128x256
    single-CTA tiles, 256x256 CTA-pair (tcgen05 cta_group::2) tiles, and clusters of two
    pairs sharing A by TMA multicast."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_10634_b200 as P
    P.lib()
    P.oz2_reset_tuning()
    assert P.oz2_set_tuning("cta_group", int(request.param[2:])) == 0
    yield P
    P.oz2_reset_tuning()


_LUT = np.array([fp8.encode_int(v) for v in range(-16, 17)], dtype=np.uint8)


def _codes_e4m3(vals):
    """Exact E4M3 codes of integers in [-16, 16] (oracle codec, vectorised by a table)."""
    v = np.asarray(vals, dtype=np.int64)
    assert v.min(initial=0) >= -16 and v.max(initial=0) <= 16
    return _LUT[v + 16]


# ------------------------------------------------------------------ raw FP8 GEMM probes

def _raw(dev, a_codes, b_codes):
    import torch
    m, k = a_codes.shape
    n = b_codes.shape[0]
    a = torch.from_numpy(np.ascontiguousarray(a_codes)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(b_codes)).cuda()
    c = torch.zeros(m * n, dtype=torch.float32, device="cuda")
    dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    assert dev.oz2_fp8_gemm_raw(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k) == 0
    torch.cuda.synchronize()
    return c.cpu().numpy().reshape(m, n)


def test_fp8_exactness_window_extremes(dev):
    """All-16 digits at k = 2^16 give exactly 2^24 (eq. error-free-FP8-matmult)."""
    k = 65536
    a = np.full((128, k), fp8.encode_int(16), dtype=np.uint8)
    a[1::2] = fp8.encode_int(-16)
    b = np.full((256, k), fp8.encode_int(16), dtype=np.uint8)
    c = _raw(dev, a, b)
    assert np.all(c[0::2] == 2.0 ** 24) and np.all(c[1::2] == -(2.0 ** 24))


@pytest.mark.parametrize("k", [32, 4096, 65536])
def test_fp8_random_digits_exact(dev, k):
    """Random integer digits in [-16, 16]: the FP32 accumulation is exact."""
    rng = np.random.default_rng(k)
    m, n = 192, 300                       # ragged: 2 x 2 tiles
    A = rng.integers(-16, 17, size=(m, k))
    B = rng.integers(-16, 17, size=(n, k))
    c = _raw(dev, _codes_e4m3(A), _codes_e4m3(B))
    want = scheme.exact_int_matmul(A, B.T)
    assert np.array_equal(c.astype(np.int64), want)


def test_fp8_bound_rounding_within_R5(dev):
    """Non-negative FP8 values across the exponent range (like A-bar B-bar): the
    tensor-core FP32 result underestimates the exact sum by < k 2^-23 (reading R5)."""
    rng = np.random.default_rng(7)
    k = 16384
    m, n = 128, 256
    codes_a = rng.integers(0x01, 0x79, size=(m, k)).astype(np.uint8)
    codes_b = rng.integers(0x01, 0x79, size=(n, k)).astype(np.uint8)
    c = _raw(dev, codes_a, codes_b)
    exactv = scheme.exact_int_matmul(scheme.fp8_scaled_int(codes_a), scheme.fp8_scaled_int(codes_b).T)
    ex = exactv.astype(np.float64) / 2.0 ** 18
    rel = (ex - c.astype(np.float64)) / ex
    assert rel.max() < k * 2.0 ** -23
    assert np.abs(rel).max() < k * 2.0 ** -23


def test_fp8_gemm_bound_entry_matches_raw(dev):
    """oz2_fp8_gemm_bound (step 2's kernel on plain operands): its row / column maxima are
    exactly the maxima of the raw FP32 accumulator of the same kernel family, ragged sizes."""
    import torch
    rng = np.random.default_rng(11)
    m, n, k = 300, 520, 2048 + 128
    codes_a = rng.integers(0x01, 0x79, size=(m, k)).astype(np.uint8)
    codes_b = rng.integers(0x01, 0x79, size=(n, k)).astype(np.uint8)
    c = _raw(dev, codes_a, codes_b)
    a = torch.from_numpy(codes_a).cuda()
    b = torch.from_numpy(codes_b).cuda()
    rmax = torch.zeros(m, dtype=torch.int32, device="cuda")
    smax = torch.zeros(n, dtype=torch.int32, device="cuda")
    assert dev.oz2_fp8_gemm_bound(a.data_ptr(), b.data_ptr(), rmax.data_ptr(), smax.data_ptr(), m, n, k) == 0
    torch.cuda.synchronize()
    r = rmax.cpu().numpy().view(np.float32)
    s = smax.cpu().numpy().view(np.float32)
    assert np.array_equal(r, c.max(axis=1)) and np.array_equal(s, c.max(axis=0))


# ------------------------------------------------------------------ full pipeline parity

def _certified_pairs(Aint, BintT, P, rows, cols):
    """Condition 2 sum_h |a'_ih||b'_hj| < P for every (i, j) with i in rows
    or j in cols, exactly in Python integers."""
    absA = np.abs(Aint.astype(object))
    absB = np.abs(BintT.astype(object))
    for i in rows:
        s = absB.dot(absA[i])                       # over all j
        assert all(2 * int(v) < P for v in s), ("row", i)
    for j in cols:
        s = absA.dot(absB[j])                       # over all i
        assert all(2 * int(v) < P for v in s), ("col", j)


def _compare(res, ref, A, B, N, family=None):
    """Stage-by-stage parity (bars in the module docstring).  Rows / columns whose GPU
    exponent differs from the oracle's own (the R6 rounding window) are not skipped: the
    oracle is re-run with the GPU's exponents (reading R13: given the exponents, the
    residues and C are unique), the certified condition is checked exactly
    for every pair they touch, and then EVERY residue and EVERY entry of C must be
    bit-exact.  Returns the mask of entries whose row and column exponents agreed."""
    if family is None:
        family = "karatsuba" if ref.plan.moduli[0] == 513 else "hybrid"
    m, n = A.shape[0], B.shape[1]
    assert res["e_prime_a"].tolist() == ref.e_prime_A
    assert res["e_prime_b"].tolist() == ref.e_prime_B
    assert np.array_equal(res["abar"], ref.Abar)
    assert np.array_equal(res["bbar"], ref.BbarT)
    # R, S: sound and close (tensor-core rounding, R5/R6)
    k = A.shape[1]
    Cx = scheme.bound_product_exact(ref.Abar, ref.BbarT).astype(np.float64) / 2.0 ** 18
    for i in range(m):
        exact_max = Cx[i].max() if n else 0.0
        g = float(res["rmax"][i])
        assert g <= exact_max * (1 + 2.0 ** -23) and g >= exact_max * (1 - k * 2.0 ** -23)
    for j in range(n):
        exact_max = Cx[:, j].max() if m else 0.0
        g = float(res["smax"][j])
        assert g <= exact_max * (1 + 2.0 ** -23) and g >= exact_max * (1 - k * 2.0 ** -23)
    rows_ok = [res["e_mu"][i] == ref.e_mu[i] for i in range(m)]
    cols_ok = [res["e_nu"][j] == ref.e_nu[j] for j in range(n)]
    # exponents may differ only where the tensor core's FP32 rounding of C-bar' moves the
    # floor of eq. mu-computation: the GPU's offset must lie between the offsets of the
    # exact maximum and of its k 2^-23 underestimate
    Pp, dlt = ref.Pp, ref.delta
    for i in range(m):
        if not rows_ok[i]:
            lo = scheme.scaling_offset(Fraction(float(Cx[i].max())) * (1 - Fraction(k, 2 ** 23)), k, Pp, dlt)
            hi = scheme.scaling_offset(Fraction(float(Cx[i].max())), k, Pp, dlt)
            assert hi <= res["e_mu"][i] - ref.e_prime_A[i] <= lo
    for j in range(n):
        if not cols_ok[j]:
            lo = scheme.scaling_offset(Fraction(float(Cx[:, j].max())) * (1 - Fraction(k, 2 ** 23)), k, Pp, dlt)
            hi = scheme.scaling_offset(Fraction(float(Cx[:, j].max())), k, Pp, dlt)
            assert hi <= res["e_nu"][j] - ref.e_prime_B[j] <= lo
    assert sum(rows_ok) >= m - 1 and sum(cols_ok) >= n - 1
    if all(rows_ok) and all(cols_ok):
        ref2 = ref
    else:
        ref2 = scheme.dgemm(A, B, N, e_mu=[int(v) for v in res["e_mu"]],
                            e_nu=[int(v) for v in res["e_nu"]], family=family)
        _certified_pairs(ref2.extra["Aint"], ref2.extra["BintT"], ref2.plan.P,
                         [i for i in range(m) if not rows_ok[i]],
                         [j for j in range(n) if not cols_ok[j]])
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref2.residues[l]), l
    assert np.array_equal(res["C"], ref2.C)
    mask = np.outer(rows_ok, cols_ok)
    assert np.array_equal(res["C"][mask], ref.C[mask])
    return mask


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_config1_64cubed_N14(dev, seed):
    """BASELINE config 1: m=n=k=64, 14 moduli, uniform [-1,1]: bit-exact residues."""
    from gpu_helpers import run
    A = gen_host(64, 64, "uniform", seed=seed)
    B = gen_host(64, 64, "uniform", seed=100 + seed)
    ref = scheme.dgemm(A, B, 14, want_digits=True)
    res = run(A, B, 14, want_digits=True)
    mask = _compare(res, ref, A, B, 14)
    assert mask.all()
    # digit planes (same tie rule R9) bit-exact
    planes_a = [pl for (da, db) in ref.extra["digits"] for pl in da]
    planes_b = [pl for (da, db) in ref.extra["digits"] for pl in db]
    for x, pl in enumerate(planes_a):
        assert np.array_equal(res["digits_a"][x], _codes_e4m3(pl)), x
    for x, pl in enumerate(planes_b):
        assert np.array_equal(res["digits_b"][x], _codes_e4m3(pl)), x
    assert res["status"] == 0


@pytest.mark.parametrize("transa,transb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("N,phi", [(12, 1.0), (13, 4.0), (7, 0.5)])
def test_ragged_layouts(dev, transa, transb, N, phi):
    """Several tiles and ragged tails in m, n and k, all four op() combinations."""
    from gpu_helpers import run
    m, k, n = 200, 300, 290
    A = gen_host(m, k, "phi", phi=phi, seed=3)
    B = gen_host(k, n, "phi", phi=phi, seed=4)
    A[5, :] = 0.0
    B[:, 7] = 0.0
    ref = scheme.dgemm(A, B, N)
    res = run(A, B, N, transa, transb, ldc_pad=3)
    mask = _compare(res, ref, A, B, N)
    assert mask.mean() > 0.98
    assert np.all(res["C_pad"] == 0.0)           # ldc padding untouched
    rel = np.linalg.norm(res["C"] - ref.C) / np.linalg.norm(ref.C)
    assert rel <= 1e-15


@pytest.mark.parametrize("N", [2, 6, 12, 16, 20, 27, 33])
def test_imported_exponents_bit_exact(dev, N):
    """Oracle exponents fed to the GPU (oracle -> GPU only): every residue and every
    output element bit-exact, including huge |A'| (>= 2^63 for N >= 14)."""
    from gpu_helpers import run
    m, k, n = 130, 257, 260
    A = gen_host(m, k, "phi", phi=2.0, seed=5)
    B = gen_host(k, n, "phi", phi=2.0, seed=6)
    ref = scheme.dgemm(A, B, N)
    res = run(A, B, N, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu)
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref.residues[l]), l
    assert np.array_equal(res["C"], ref.C)


_SCHED_REF = {}


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("sch", ["fp8", "int8"])
def test_work_item_schedules(dev, split, sch, knobs):
    """Both residue-GEMM schedules -- tile-major (every modulus of a tile in one work item,
    CRT fused into the epilogue for k >= 8192) and modulus-split (one (tile, modulus) item,
    separate CRT; automatic for grids with few tiles) -- give the oracle's residues and C
    bit for bit (imported exponents), with alpha/beta and k >= 8192."""
    from gpu_helpers import run
    from oracle import int8
    knobs(mod_split=split, fused_crt=1)             # tile-major then fuses (k >= 8192)
    m, k, n, N = 16, 8200, 24, 13
    A = gen_host(m, k, "phi", phi=1.0, seed=51)
    B = gen_host(k, n, "phi", phi=1.0, seed=52)
    if sch not in _SCHED_REF:
        _SCHED_REF[sch] = int8.dgemm(A, B, N) if sch == "int8" else scheme.dgemm(A, B, N)
    ref = _SCHED_REF[sch]
    res = run(A, B, N, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu, scheme=sch, alpha=2.0, beta=0.5,
              C0=np.ones((m, n)))
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref.residues[l]), l
    want = np.array([[float(Fraction(2) * Fraction(float(ref.C[i, j])) + Fraction(0.5))
                      for j in range(n)] for i in range(m)])
    assert np.array_equal(res["C"], want)


@pytest.mark.parametrize("sch", ["fp8", "int8", "karatsuba"])
def test_work_item_schedules_agree_many_tiles(dev, sch, knobs):
    """Tile-major (fused CRT) and modulus-split schedules on a grid of 4 x 5 CTA-pair tiles
    with ragged edges: identical residues and C (both are exact), and the oracle's on one
    sampled entry per tile (exponents, residues and C, tests/sampled.py)."""
    from gpu_helpers import run
    m, k, n, N = 1000, 8192, 1100, 14
    A = gen_host(m, k, "phi", phi=2.0, seed=53)
    B = gen_host(k, n, "phi", phi=2.0, seed=54)
    outs = []
    for split in ["0", "1"]:
        knobs(fused_crt=1, mod_split=split)        # tile-major then fuses (k >= 8192)
        outs.append(run(A, B, N, scheme=sch))
    knobs(fused_crt=0, mod_split=0)                # tile-major with the separate CRT
    outs.append(run(A, B, N, scheme=sch))
    assert np.array_equal(outs[0]["C"], outs[2]["C"])
    knobs(mod_split=2)                             # hybrid: full waves tile-major, tail split
    outs.append(run(A, B, N, scheme=sch))
    assert np.array_equal(outs[0]["residues"], outs[3]["residues"])
    assert np.array_equal(outs[0]["C"], outs[3]["C"])
    assert np.array_equal(outs[0]["e_mu"], outs[1]["e_mu"])
    assert np.array_equal(outs[0]["residues"], outs[1]["residues"])
    assert np.array_equal(outs[0]["C"], outs[1]["C"])
    from sampled import check_sampled, col_cover, tile_cover
    I, J = tile_cover(m), col_cover(n)
    o = outs[0]
    gpu = {"e_mu": o["e_mu"], "e_nu": o["e_nu"], "C": o["C"][np.ix_(I, J)],
           "res": np.array([R[np.ix_(I, J)] for R in o["residues"]])}
    fam = {"fp8": "hybrid", "int8": "int8", "karatsuba": "karatsuba"}[sch]
    check_sampled(A, B, N, I, J, gpu, family=fam, accuracy=False)


def test_alpha_beta_and_quick_returns(dev):
    from gpu_helpers import run
    m, k, n = 70, 90, 80
    A = gen_host(m, k, "phi", phi=1.0, seed=8)
    B = gen_host(k, n, "phi", phi=1.0, seed=9)
    C0 = gen_host(m, n, "uniform", seed=10)
    ref = scheme.dgemm(A, B, 12, alpha=-1.5, beta=0.25, C=C0)
    res = run(A, B, 12, alpha=-1.5, beta=0.25, C0=C0)
    assert np.array_equal(res["C"], ref.C)
    res0 = run(A, B, 12, alpha=0.0, beta=2.0, C0=C0)
    assert np.array_equal(res0["C"], 2.0 * C0)
    Ak = np.zeros((m, 0))
    Bk = np.zeros((0, n))
    resk = run(Ak, Bk, 12, alpha=1.0, beta=0.0, C0=C0)
    assert np.all(resk["C"] == 0.0)


def test_identity_and_integer_exact(dev):
    from gpu_helpers import run
    I = np.eye(40)
    assert np.array_equal(run(I, I, 12)["C"], I)
    A = gen_host(16, 64, "int", seed=1)
    B = gen_host(64, 16, "int", seed=2)
    want = (A.astype(object).dot(B.astype(object))).astype(np.float64)
    assert np.array_equal(run(A, B, 12)["C"], want)


@pytest.mark.parametrize("sch,mode", [("fp8", "accurate"), ("fp8", "fast"), ("int8", "accurate")])
def test_nonfinite_status(dev, sch, mode):
    """Reading R12: a NaN / Inf in row i of A (column j of B) sets the status word and
    makes row i (column j) of C NaN; every other entry stays finite."""
    from gpu_helpers import run
    A = gen_host(20, 30, "uniform", seed=1)
    B = gen_host(30, 10, "uniform", seed=2)
    A[3, 4] = np.nan
    B[7, 6] = np.inf
    res = run(A, B, 12, scheme=sch, mode=mode)
    assert res["status"] == dev.OZ2_ERR_NONFINITE
    C = res["C"]
    assert np.all(np.isnan(C[3, :])) and np.all(np.isnan(C[:, 6]))
    mask = np.ones(C.shape, dtype=bool)
    mask[3, :] = False
    mask[:, 6] = False
    assert np.all(np.isfinite(C[mask]))


def test_host_pointer_path(dev):
    """Host (numpy) buffers through the same C ABI give the same bits as device ones."""
    from gpu_helpers import run
    m, k, n = 150, 200, 170
    A = np.asfortranarray(gen_host(m, k, "phi", phi=1.0, seed=11))
    B = np.asfortranarray(gen_host(k, n, "phi", phi=1.0, seed=12))
    C = np.asfortranarray(np.zeros((m, n)))
    rc = dev.oz2_dgemm("N", "N", m, n, k, 1.0, A.ctypes.data, m, B.ctypes.data, k, 0.0, C.ctypes.data, m, 13)
    assert rc == 0
    assert np.array_equal(C, run(A, B, 13)["C"])


@pytest.mark.parametrize("blocks,pinned", [("1", True), ("4", True), ("3", True), ("4", False)])
def test_host_pointer_column_blocks(dev, blocks, pinned, knobs):
    """Host buffers with C returned in column blocks (each block's device-to-host copy
    overlaps the next block's GEMMs; OZ2_TUNE_HOST_BLOCKS, pinned C only -- pageable C is
    copied in one piece): bit-identical to the device-pointer call, including a ragged
    last block, ldc padding, beta != 0 and transposed A."""
    import torch
    from gpu_helpers import run
    knobs(host_blocks=blocks)
    m, k, n = 300, 260, 2600
    A = gen_host(m, k, "phi", phi=1.0, seed=21)
    B = gen_host(k, n, "phi", phi=1.0, seed=22)
    C0 = gen_host(m, n, "uniform", seed=23)
    At = np.asfortranarray(A.T)                       # op(A) = A with transa = 'T'
    Bh = np.asfortranarray(B)
    ldc = m + 5
    if pinned:
        Ch = torch.zeros((n, ldc), dtype=torch.float64, pin_memory=True).numpy().T
    else:
        Ch = np.asfortranarray(np.zeros((ldc, n)))
    Ch[:m] = C0
    rc = dev.oz2_dgemm("T", "N", m, n, k, 0.5, At.ctypes.data, k, Bh.ctypes.data, k, -1.5,
                       Ch.ctypes.data, ldc, 13)
    assert rc == 0
    ref = run(A, B, 13, alpha=0.5, beta=-1.5, C0=C0)["C"]
    assert np.array_equal(Ch[:m], ref)
    assert np.all(Ch[m:] == 0.0)


def test_per_call_options(dev):
    """oz2_options.set_mode / set_scheme apply to one call only and equal the thread-level
    setting; timing_ms receives the phase times (total = sum of the phases)."""
    import ctypes
    import torch
    m, k, n = 300, 400, 260
    A = torch.from_numpy(gen_host(m, k, "phi", phi=1.0, seed=15)).cuda()
    B = torch.from_numpy(gen_host(k, n, "phi", phi=1.0, seed=16)).cuda()
    A = A.t().contiguous().t()
    B = B.t().contiguous().t()
    outs = {}
    for mode, sch in [("fast", "fp8"), ("accurate", "int8"), ("fast", "karatsuba")]:
        C1 = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        C2 = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        opt = dev.oz2_options()
        opt.set_mode, opt.mode = 1, {"accurate": 0, "fast": 1}[mode]
        opt.set_scheme, opt.scheme = 1, {"fp8": 0, "int8": 1, "karatsuba": 2}[sch]
        ms = (ctypes.c_float * 7)()
        opt.timing_ms = ctypes.addressof(ms)
        dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
        dev.oz2_set_workspace(None, 0)
        assert dev.oz2_dgemm_ex("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                                C1.data_ptr(), m, 14, opt) == 0
        assert dev.oz2_get_mode() == 0 and dev.oz2_get_scheme() == 0     # thread settings untouched
        assert ms[6] > 0 and abs(sum(ms[:6]) - ms[6]) < 0.05 * ms[6] + 0.05
        dev.oz2_set_mode(mode)
        dev.oz2_set_scheme(sch)
        try:
            assert dev.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                                 C2.data_ptr(), m, 14) == 0
        finally:
            dev.oz2_set_mode("accurate")
            dev.oz2_set_scheme("fp8")
        torch.cuda.synchronize()
        assert torch.equal(C1, C2)
        outs[(mode, sch)] = C1
    assert not torch.equal(outs[("fast", "fp8")], outs[("fast", "karatsuba")])
    bad = dev.oz2_options()
    bad.set_mode, bad.mode = 1, 7
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    assert dev.oz2_dgemm_ex("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                            C.data_ptr(), m, 14, bad) == -15


def test_torch_wrapper_strided_C(dev):
    """dgemm() into a non-contiguous view (every other column of a larger matrix): the
    other columns stay untouched and the view gets the same C as a dense call."""
    import torch
    A = torch.from_numpy(gen_host(70, 90, "phi", phi=1.0, seed=17)).cuda()
    B = torch.from_numpy(gen_host(90, 40, "phi", phi=1.0, seed=18)).cuda()
    big = torch.full((70, 80), 7.0, dtype=torch.float64, device="cuda")
    view = big[:, ::2]
    dev.dgemm(A, B, C=view, num_moduli=13)
    ref = dev.dgemm(A, B, num_moduli=13)
    assert torch.equal(view, ref)
    assert torch.all(big[:, 1::2] == 7.0)
    C0 = torch.from_numpy(gen_host(70, 40, "uniform", seed=19)).cuda()
    big2 = torch.zeros((80, 70), dtype=torch.float64, device="cuda").t()[:, :40]   # col-major, ld 70
    big2.copy_(C0)
    dev.dgemm(A, B, alpha=2.0, beta=-1.0, C=big2, num_moduli=13)
    big3 = torch.zeros((40, 140), dtype=torch.float64, device="cuda").t()[::2]      # stride (2, 140)
    big3.copy_(C0)
    dev.dgemm(A, B, alpha=2.0, beta=-1.0, C=big3, num_moduli=13)
    assert torch.equal(big2, big3)


def test_torch_wrapper_layouts(dev):
    import torch
    A = torch.from_numpy(gen_host(100, 120, "phi", phi=1.0, seed=13, order="C")).cuda()
    B = torch.from_numpy(gen_host(120, 90, "phi", phi=1.0, seed=14, order="C")).cuda()
    C1 = dev.dgemm(A, B, num_moduli=13)
    C2 = dev.dgemm(A.t().contiguous().t(), B.t().contiguous().t(), num_moduli=13)
    ref = A @ B
    assert torch.equal(C1, C2)
    assert (torch.linalg.norm(C1 - ref) / torch.linalg.norm(ref)).item() < 1e-14
    C3 = torch.zeros(100, 90, dtype=torch.float64, device="cuda")     # row-major C
    dev.dgemm(A, B, C=C3, num_moduli=13)
    assert (torch.linalg.norm(C3 - ref) / torch.linalg.norm(ref)).item() < 1e-14


def test_workspace_and_timing_api(dev):
    """Caller-owned workspace (below the full size -> m/n blocking, far too small ->
    OZ2_ERR_WORKSPACE, exact size works unblocked), the per-phase timers, and the
    single-process path of the row-sharded driver."""
    import torch
    from paper_2603_10634_b200.dist import dgemm_rowsharded
    m, k, n, N = 300, 520, 270, 13
    A = torch.from_numpy(gen_host(m, k, "phi", phi=1.0, seed=51)).cuda()
    B = torch.from_numpy(gen_host(k, n, "phi", phi=1.0, seed=52)).cuda()
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    need = dev.oz2_workspace_size("N", "N", m, n, k, N)
    small = torch.empty(need - 1024, dtype=torch.uint8, device="cuda")
    dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    dev.oz2_set_workspace(small.data_ptr(), small.numel())
    args = ("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, N)
    assert dev.oz2_dgemm(*args) == 0
    assert dev.oz2_get_blocking() != (m, n)
    torch.cuda.synchronize()
    C_blocked = C.cpu().numpy().copy()
    dev.oz2_set_workspace(small.data_ptr(), 4096)
    assert dev.oz2_dgemm(*args) == dev.OZ2_ERR_WORKSPACE
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    dev.oz2_set_workspace(ws.data_ptr(), ws.numel())
    dev.oz2_set_timing(True)
    assert dev.oz2_dgemm(*args) == 0
    ph = dev.oz2_get_timing()
    dev.oz2_set_timing(False)
    assert set(ph) == set(dev.PHASES)
    parts = sum(v for key, v in ph.items() if key != "total")
    assert ph["total"] > 0 and abs(parts - ph["total"]) <= 0.05 * ph["total"] + 0.05
    dev.oz2_set_workspace(None, 0)
    assert dev.oz2_get_blocking() == (m, n)
    ref = scheme.dgemm(A.cpu().numpy(), B.cpu().numpy(), N).C
    assert np.array_equal(C.cpu().numpy(), ref)
    assert np.array_equal(C_blocked, ref)
    C2 = dgemm_rowsharded(A, B, num_moduli=N)          # no process group: plain call
    assert np.array_equal(C2.cpu().numpy(), ref)


_LONGK_REF = {}


@pytest.mark.parametrize("fam", ["hybrid", "karatsuba"])
@pytest.mark.parametrize("sched", ["split", "tile_fused"])
def test_k_beyond_exactness_window(dev, fam, sched, knobs):
    """k > 2^16 (NEXT-2): products run in 2^16-long K segments reduced mod p; residues and C
    stay bit-exact against the oracle, which needs no segmentation (exact integers) -- for
    both FP8 families and both work-item schedules (tile-major with the fused CRT)."""
    from gpu_helpers import run
    m, k, n, N = 16, 65536 + 300, 24, 12 if fam == "hybrid" else 13
    if sched == "tile_fused":
        knobs(mod_split=0, fused_crt=1)
    A = gen_host(m, k, "phi", phi=1.0, seed=61)
    B = gen_host(k, n, "phi", phi=1.0, seed=62)
    if fam not in _LONGK_REF:
        _LONGK_REF[fam] = scheme.dgemm(A, B, N, family=fam)
    ref = _LONGK_REF[fam]
    res = run(A, B, N, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu, scheme="fp8" if fam == "hybrid" else "karatsuba")
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref.residues[l]), l
    assert np.array_equal(res["C"], ref.C)


def _depth_edge_matrix(pmin, m=24, k=160, seed=0):
    """Rows whose largest |entry| sits just below / at / above the reduction-depth limits
    2^50 p_min and 2^86 p_min of the residue kernel (and far beyond), as exact integers."""
    rng = np.random.default_rng(seed)
    A = rng.integers(-1000, 1000, size=(m, k)).astype(np.float64)
    lim1, lim2 = float(pmin) * 2.0 ** 50, float(pmin) * 2.0 ** 86
    edges = [lim1 - 2 ** 12, lim1, lim1 + 2 ** 12, lim2 * (1 - 2.0 ** -40), lim2, lim2 * (1 + 2.0 ** -40),
             2.0 ** 63 - 2 ** 11, 2.0 ** 64, 2.0 ** 96 - 2.0 ** 44, 2.0 ** 120 + 2.0 ** 70]
    for i, v in enumerate(edges):
        A[2 * i, 3 + i] = v
        A[2 * i + 1, 5 + i] = -v
        A[2 * i + 1, 7 + i] = np.floor(v / 3)
    return A


@pytest.mark.parametrize("sch,N", [("fp8", 12), ("fp8", 20), ("fp8", 33), ("int8", 15), ("int8", 33)])
def test_residue_depth_boundaries(dev, sch, N):
    """Imported zero exponents make A' = A: residues of integers straddling every
    reduction-depth switch of k_digits must match mod(A'B', p) exactly (CRT output not
    compared: the certified condition is deliberately violated)."""
    from gpu_helpers import run
    from oracle import moduli as mod
    ps = mod.int8_moduli(N) if sch == "int8" else mod.hybrid_moduli(N)
    A = _depth_edge_matrix(min(ps), seed=N)
    rng = np.random.default_rng(N + 1)
    B = rng.integers(-1000, 1000, size=(A.shape[1], 40)).astype(np.float64)
    res = run(A, B, N, e_mu_in=[0] * A.shape[0], e_nu_in=[0] * B.shape[1], scheme=sch)
    Aint = scheme.to_integral(A, [0] * A.shape[0])
    BintT = scheme.to_integral(B.T.copy(), [0] * B.shape[1])
    for l, p in enumerate(ps):
        want = scheme.modprod_direct(scheme.residues(Aint, p), scheme.residues(BintT, p), p)
        assert np.array_equal(res["residues"][l], want), p


@pytest.mark.parametrize("sch", ["fp8", "int8"])
def test_cuda_graph_capture(dev, sch):
    """After a first call has built the plan and the workspace, oz2_dgemm only enqueues
    asynchronous work on the library's stream, so it can be captured in a CUDA graph and
    replayed (small shapes are launch-bound); replays give the direct call's bits."""
    import torch
    m, k, n, N = 384, 1000, 520, 13
    A = torch.from_numpy(np.asfortranarray(gen_host(m, k, "phi", phi=1.0, seed=71))).cuda()
    B = torch.from_numpy(np.asfortranarray(gen_host(k, n, "phi", phi=1.0, seed=72))).cuda()
    Ad = A.t().contiguous().t()           # column-major storage
    Bd = B.t().contiguous().t()
    C_ref = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    C_g = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    assert dev.oz2_set_scheme(sch) == 0
    try:
        ws = torch.empty(dev.oz2_workspace_size("N", "N", m, n, k, N), dtype=torch.uint8, device="cuda")
        dev.oz2_set_workspace(ws.data_ptr(), ws.numel())
        call = lambda C: dev.oz2_dgemm("N", "N", m, n, k, 1.0, Ad.data_ptr(), m, Bd.data_ptr(), k, 0.0,
                                       C.data_ptr(), m, N)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            dev.oz2_set_stream(s.cuda_stream)
            assert call(C_ref) == 0                     # warm-up: plan + device constants
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
            assert call(C_g) == 0
        for _ in range(3):
            C_g.zero_()
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C_g, C_ref)
    finally:
        dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
        dev.oz2_set_workspace(None, 0)
        dev.oz2_set_scheme("fp8")


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (1, 257, 1), (300, 1, 2), (2, 3, 1), (1, 5000, 3), (257, 2, 255)])
@pytest.mark.parametrize("sch", ["fp8", "int8", "karatsuba"])
def test_degenerate_shapes(dev, m, k, n, sch):
    """Vectors, k = 1 and sub-tile shapes: residues and C bit-exact against the oracle
    (imported exponents, so the R6 rounding window cannot intervene)."""
    from gpu_helpers import run
    from oracle import int8
    A = gen_host(m, k, "phi", phi=1.5, seed=m + 7 * k)
    B = gen_host(k, n, "phi", phi=1.5, seed=n + 11 * k)
    N = 13
    ref = (int8.dgemm(A, B, N) if sch == "int8"
           else scheme.dgemm(A, B, N, family="karatsuba" if sch == "karatsuba" else "hybrid"))
    res = run(A, B, N, e_mu_in=ref.e_mu, e_nu_in=ref.e_nu, scheme=sch)
    for l in range(N):
        assert np.array_equal(res["residues"][l], ref.residues[l]), l
    assert np.array_equal(res["C"], ref.C)


def test_concurrent_host_threads(dev):
    """The library state (stream, workspace, scheme, plans) is per host thread: two threads
    running different schemes on their own streams at the same time get the bits of the
    sequential calls."""
    import threading
    import torch
    m, k, n = 700, 900, 600
    A = torch.from_numpy(np.asfortranarray(gen_host(m, k, "phi", phi=1.0, seed=81))).cuda()
    B = torch.from_numpy(np.asfortranarray(gen_host(k, n, "phi", phi=1.0, seed=82))).cuda()
    Ad, Bd = A.t().contiguous().t(), B.t().contiguous().t()

    def call(scheme, N, out):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            dev.oz2_set_stream(s.cuda_stream)
            assert dev.oz2_set_scheme(scheme) == 0
            for _ in range(3):
                rc = dev.oz2_dgemm("N", "N", m, n, k, 1.0, Ad.data_ptr(), m, Bd.data_ptr(), k, 0.0,
                                   out.data_ptr(), m, N)
                assert rc == 0
            s.synchronize()
            dev.oz2_set_scheme("fp8")
            dev.oz2_finalize()

    jobs = [("fp8", 13), ("int8", 15), ("karatsuba", 14)]
    seq = [torch.empty((n, m), dtype=torch.float64, device="cuda").t() for _ in jobs]
    par = [torch.empty((n, m), dtype=torch.float64, device="cuda").t() for _ in jobs]
    for (sch, N), o in zip(jobs, seq):
        call(sch, N, o)
    errors = []

    def guarded(*a):
        try:
            call(*a)
        except BaseException as e:      # surfaced below: a thread's assert must fail the test
            errors.append(e)

    threads = [threading.Thread(target=guarded, args=(sch, N, o)) for (sch, N), o in zip(jobs, par)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    assert not errors, errors
    for a, b in zip(seq, par):
        assert torch.equal(a, b)


_CG_SNIPPET = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device
sch = sys.argv[1]
m, n, k = 2560, 2560, 1024          # 100 CTA-pair tiles: hybrid = 74 tile-major + a split tail
A = gen_device(m, k, "phi", phi=1.0, seed=91)
B = gen_device(k, n, "phi", phi=1.0, seed=92)
C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
assert P.oz2_set_scheme(sch) == 0
assert P.oz2_set_tuning("cta_group", int(sys.argv[2].rstrip("w"))) == 0
if sys.argv[2].endswith("w"):      # 256 x 512 CTA-pair tiles (FP8 kinds; INT8 keeps 256)
    assert P.oz2_set_tuning("tile_n", 512) == 0
for split in ("0", "1", "2"):
    assert P.oz2_set_tuning("mod_split", int(split)) == 0
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, 13) == 0
    torch.cuda.synchronize()
    print(split, hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest())
"""


@pytest.mark.parametrize("sch", ["fp8", "int8", "karatsuba"])
def test_gemm_variants_identical(dev, sch):
    """CTA group 1 (128x256 CTAs), 2 (CTA pairs, default), 4 (two pairs multicasting A; FP8
    kinds only, INT8 falls back to pairs), 2 with 256x512 tiles (OZ2_TUNE_TILE_N = 512; FP8
    kinds, K-concatenated square products at this k) give identical C under all three work-item
    schedules, and that C is the oracle's on one sampled entry per 256 x 256 tile.  Each
    variant runs in a subprocess with a timeout, so a pipeline hang fails the test."""
    import hashlib
    import os
    import subprocess
    import sys
    import torch
    from sampled import check_sampled, col_cover, tile_cover
    from synth import gen_device
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for cg in ["1", "2", "4", "2w"]:
        r = subprocess.run([sys.executable, "-c", _CG_SNIPPET, sch, cg], cwd=root,
                           capture_output=True, text=True, timeout=240)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[cg] = r.stdout.split()
    assert outs["1"] == outs["2"] == outs["4"] == outs["2w"]
    assert outs["2"][1] == outs["2"][3] == outs["2"][5]   # tile-major, split and hybrid agree
    # the same problem in-process (default kernels) with exponent outputs -> the oracle
    m, n, k = 2560, 2560, 1024
    A = gen_device(m, k, "phi", phi=1.0, seed=91)
    B = gen_device(k, n, "phi", phi=1.0, seed=92)
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    e_mu = torch.zeros(m, dtype=torch.int32, device="cuda")
    e_nu = torch.zeros(n, dtype=torch.int32, device="cuda")
    opt = dev.oz2_options()
    opt.e_mu, opt.e_nu = e_mu.data_ptr(), e_nu.data_ptr()
    opt.set_scheme, opt.scheme = 1, {"fp8": 0, "int8": 1, "karatsuba": 2}[sch]
    dev.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
    dev.oz2_set_workspace(None, 0)
    assert dev.oz2_dgemm_ex("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                            C.data_ptr(), m, 13, opt) == 0
    torch.cuda.synchronize()
    Ch = C.cpu().numpy()
    assert hashlib.sha256(Ch.tobytes()).hexdigest() == outs["2"][1]
    I, J = tile_cover(m), col_cover(n)
    fam = {"fp8": "hybrid", "int8": "int8", "karatsuba": "karatsuba"}[sch]
    check_sampled(A.cpu().numpy(), B.cpu().numpy(), 13, I, J,
                  {"e_mu": e_mu.cpu().numpy(), "e_nu": e_nu.cpu().numpy(), "C": Ch[np.ix_(I, J)]},
                  family=fam, accuracy=False)


@pytest.mark.parametrize("ea,eb", [(-600, -400), (500, 500), (-1030, 1000)])
def test_extreme_exponent_ranges(dev, ea, eb):
    """Inputs far from 1 (rows of A scaled by 2^ea, columns of B by 2^eb, including
    subnormal A entries for ea = -1030): the power-of-two pre/post scaling stays exact, so
    exponents, residues and C match the oracle bit for bit (results stay normal binary64)."""
    from gpu_helpers import run
    m, k, n = 40, 300, 30
    A = gen_host(m, k, "phi", phi=1.0, seed=97) * 2.0 ** ea
    B = gen_host(k, n, "phi", phi=1.0, seed=98) * 2.0 ** eb
    ref = scheme.dgemm(A, B, 13)
    res = run(A, B, 13)
    mask = _compare(res, ref, A, B, 13)
    assert mask.all()
    assert np.all(np.isfinite(res["C"]))


@pytest.mark.parametrize("k", [32768, 32763, 1000])
def test_kcat_cross_products_exactness_edge(dev, k, knobs):
    """K-concatenated square-modulus cross products (OZ2_TUNE_KCAT): A1 B2 + A2 B1
    accumulate in ONE FP32 accumulator.  Integer inputs 544 = 16 * 33 + 16 give the digits
    D1 = D2 = 16 for p = 1089, so at k = 2^15 the concatenated sum is exactly 2 k 2^8 =
    2^24, the edge of the exactness window (eq. error-free-FP8-matmult).  Residues and C
    equal the oracle's (imported exponents 0) with the concatenation on and off."""
    from gpu_helpers import run
    m, n, N = 40, 48, 13
    rng = np.random.default_rng(k)
    A = np.full((m, k), 544.0)
    B = np.full((k, n), 544.0)
    A[1::2] *= -1.0
    B[:, ::3] *= -1.0
    A[5:9] = rng.integers(-2 ** 20, 2 ** 20, size=(4, k))        # generic rows too
    B[:, 7:11] = rng.integers(-2 ** 20, 2 ** 20, size=(k, 4))
    e0 = [0] * m
    f0 = [0] * n
    I, J = list(range(m)), list(range(n))
    res_ref, C_ref = scheme.entries(A, B, N, I, J, e0, f0)
    outs = []
    for kc in (1, 0):
        knobs(kcat=kc)
        out = run(A, B, N, e_mu_in=e0, e_nu_in=f0)
        assert np.array_equal(np.array(out["residues"]), res_ref)
        assert np.array_equal(out["C"], C_ref)
        outs.append(out)
    assert np.array_equal(outs[0]["C"], outs[1]["C"])


@pytest.mark.parametrize("sch", ["fp8", "karatsuba"])
def test_kcat_on_off_identical_many_tiles(dev, sch, knobs):
    """The concatenated and the three-product forms give identical residues and C on a
    multi-tile problem through the full pipeline (k = 8192, both work-item schedules)."""
    from gpu_helpers import run
    m, k, n, N = 700, 8192, 600, 13
    A = gen_host(m, k, "phi", phi=1.0, seed=71)
    B = gen_host(k, n, "phi", phi=1.0, seed=72)
    outs = []
    for kc, split in [(1, 0), (0, 0), (1, 1)]:
        knobs(kcat=kc, mod_split=split)
        outs.append(run(A, B, N, scheme=sch))
    for o in outs[1:]:
        assert np.array_equal(o["residues"], outs[0]["residues"])
        assert np.array_equal(o["C"], outs[0]["C"])


_W512_SNIPPET = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device
sch, m, n, k, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
A = gen_device(m, k, "phi", phi=1.0, seed=93)
B = gen_device(k, n, "phi", phi=1.0, seed=94)
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
assert P.oz2_set_scheme(sch) == 0
for tn in (256, 512):
    assert P.oz2_set_tuning("tile_n", tn) == 0
    for fused in (-1, 0):
        assert P.oz2_set_tuning("fused_crt", fused) == 0
        C = torch.full((n, m), 7.0, dtype=torch.float64, device="cuda").t()
        res = torch.zeros(N * m * n, dtype=torch.int16, device="cuda")
        opt = P.oz2_options()
        opt.residues = res.data_ptr()
        assert P.oz2_dgemm_ex("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0,
                              C.data_ptr(), m, N, opt) == 0
        torch.cuda.synchronize()
        h = hashlib.sha256(C.cpu().numpy().tobytes() + res.cpu().numpy().tobytes()).hexdigest()
        print(tn, fused, h)
"""


@pytest.mark.parametrize("sch,m,n,k,N", [
    ("fp8", 1000, 1300, 16500, 13),      # fused CRT (k >= 16384), ragged m, n, k; last R half partly outside n
    ("fp8", 520, 700, 70000, 12),        # two 2^16 K segments per product
    ("karatsuba", 777, 1536, 16384, 13),
    ("fp8", 300, 2000, 1500, 20),        # K-concatenated square products (k <= 2048), 6-limb CRT
])
def test_tile_n512_identical(sch, m, n, k, N):
    """256 x 512 CTA-pair tiles (OZ2_TUNE_TILE_N = 512) give the same residues and C as the
    default 256 x 256 tiles, bit for bit, with the fused and the separate CRT (the default
    tiles are pinned to the oracle by the tests above).  Subprocess with a timeout: a
    pipeline hang fails the test instead of blocking the suite."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _W512_SNIPPET, sch, str(m), str(n), str(k), str(N)],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln.split() for ln in r.stdout.strip().splitlines()]
    assert len(lines) == 4
    assert len({ln[2] for ln in lines}) == 1, lines


_CANARY_SNIPPET = r"""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device
ta, tb, m, n, k, N, sch, mode, tile_n, blocked = sys.argv[1], sys.argv[2], *map(int, sys.argv[3:7]), sys.argv[7], sys.argv[8], int(sys.argv[9]), int(sys.argv[10])
A = gen_device(m, k, "phi", phi=1.0, seed=71)
B = gen_device(k, n, "phi", phi=1.0, seed=72)
Ast, lda = (A.t().contiguous().t(), m) if ta == "N" else (A.contiguous(), k)
Bst, ldb = (B.t().contiguous().t(), k) if tb == "N" else (B.contiguous(), n)
ldc = m + 5
Cbuf = torch.full((n, ldc), 3.25, dtype=torch.float64, device="cuda")
assert P.oz2_set_scheme(sch) == 0 and P.oz2_set_mode(mode) == 0
assert P.oz2_set_tuning("tile_n", tile_n) == 0
need = P.oz2_workspace_size(ta, tb, m, n, k, N)
if blocked:                                 # a third of the unblocked workspace: m/n blocking
    need = need // 3
GUARD = 1 << 20
ws = torch.full((need + 2 * GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
P.oz2_set_workspace(ws.data_ptr() + GUARD, need)
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
a0, b0 = Ast.clone(), Bst.clone()
rc = P.oz2_dgemm(ta, tb, m, n, k, 1.0, Ast.data_ptr(), lda, Bst.data_ptr(), ldb, 0.0, Cbuf.data_ptr(), ldc, N)
torch.cuda.synchronize()
assert rc == 0, rc
assert bool((ws[:GUARD] == 0xA5).all()), "workspace head guard written"
assert bool((ws[GUARD + need:] == 0xA5).all()), "workspace tail guard written"
assert torch.equal(Ast, a0) and torch.equal(Bst, b0), "inputs modified"
assert bool((Cbuf[:, m:] == 3.25).all()), "ldc padding written"
C = Cbuf[:, :m].t()
ref = A @ B
rel = (torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item()
assert rel < 1e-14, rel
print("ok", rel)
"""


@pytest.mark.parametrize("ta,tb,m,n,k,N,sch,mode,tile_n,blocked", [
    ("N", "N", 300, 260, 701, 13, "fp8", "accurate", 256, 0),     # k_cast MN-major / K-major (odd ld: scalar loads)
    ("T", "T", 300, 260, 701, 13, "fp8", "accurate", 256, 0),
    ("T", "N", 300, 260, 2300, 13, "fp8", "accurate", 256, 0),    # 16-byte K-major loads, 2 super-chunks
    ("N", "T", 300, 260, 701, 13, "fp8", "fast", 256, 0),         # sums of squares
    ("T", "N", 300, 260, 701, 15, "int8", "accurate", 256, 0),
    ("N", "N", 520, 700, 16500, 13, "fp8", "accurate", 512, 0),   # 256 x 512 tiles, fused CRT
    ("N", "N", 1000, 900, 3000, 13, "fp8", "accurate", 256, 1),   # m/n blocking
])
def test_workspace_and_buffer_guards(ta, tb, m, n, k, N, sch, mode, tile_n, blocked):
    """Bounds check of our own (compute-sanitizer is not available on the GPU pool): 1 MiB
    guard bands of 0xA5 before and after a caller workspace of exactly the required size
    stay untouched, the inputs are unmodified, the ldc padding of C is not written, and C
    is accurate -- over the storage orders, odd / even k (scalar / vector loads of the
    cast), fast mode, the INT8 scheme, 256 x 512 tiles and m/n blocking."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    args = [ta, tb, str(m), str(n), str(k), str(N), sch, mode, str(tile_n), str(blocked)]
    r = subprocess.run([sys.executable, "-c", _CANARY_SNIPPET, *args], cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout + r.stderr)[-2000:]
    assert r.stdout.startswith("ok")


_HYBRID_SNIPPET = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2603_10634_b200 as P
from synth import gen_device
sch, cg, tile_n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
m, n, k, N = 2560, 2560, 16384, 13 if sch != "int8" else 15
A = gen_device(m, k, "phi", phi=1.0, seed=81)
B = gen_device(k, n, "phi", phi=1.0, seed=82)
C0 = gen_device(m, n, "uniform", seed=83)
P.oz2_set_stream(torch.cuda.current_stream().cuda_stream)
assert P.oz2_set_scheme(sch) == 0
assert P.oz2_set_tuning("cta_group", cg) == 0 and P.oz2_set_tuning("tile_n", tile_n) == 0
for split, fused in ((0, 1), (2, 1), (2, 0), (1, 0)):
    assert P.oz2_set_tuning("mod_split", split) == 0 and P.oz2_set_tuning("fused_crt", fused) == 0
    C = C0.clone()
    assert P.oz2_dgemm("N", "N", m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.5, C.data_ptr(), m, N) == 0
    torch.cuda.synchronize()
    print(split, fused, hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest())
"""


@pytest.mark.parametrize("sch,cg,tile_n", [("fp8", 2, 256), ("fp8", 1, 256), ("fp8", 4, 256),
                                           ("fp8", 2, 512), ("karatsuba", 2, 256), ("int8", 2, 256)])
def test_hybrid_schedule_with_fused_crt(sch, cg, tile_n):
    """The hybrid schedule with the fused CRT (tile-major head items keep the CRT in the
    GEMM epilogue, the split tail's tiles get theirs from k_crt_tiles) gives the same C as
    tile-major + fused, hybrid + separate CRT and all-split, bit for bit, with beta != 0 (a
    tile whose CRT ran twice would apply beta twice).  2560^2 x 16384: 100 CTA-pair tiles,
    74 in the head wave, a 26-tile tail.  Subprocess with a timeout."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _HYBRID_SNIPPET, sch, str(cg), str(tile_n)], cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln.split() for ln in r.stdout.strip().splitlines()]
    assert len(lines) == 4
    assert len({ln[2] for ln in lines}) == 1, lines
