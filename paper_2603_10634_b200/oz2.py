"""Python binding of liboz2.so (include/oz2.h) -- argument marshalling only.

Every step of the emulation runs in the library's CUDA kernels; this module only
loads the shared library with ctypes, declares the C signatures and converts
arguments.  There is no CPU fallback: if liboz2.so is missing or no sm_100 device
is present the calls fail loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboz2.so")

OZ2_SUCCESS = 0
OZ2_ERR_CUDA = 1
OZ2_ERR_ALLOC = 2
OZ2_ERR_WORKSPACE = 3
OZ2_ERR_NOT_SUPPORTED = 4
OZ2_ERR_NONFINITE = 5
OZ2_SCHEME_FP8 = 0
OZ2_SCHEME_INT8 = 1
OZ2_SCHEME_FP8_KARATSUBA = 2
_SCHEMES = {"fp8": OZ2_SCHEME_FP8, "int8": OZ2_SCHEME_INT8, "karatsuba": OZ2_SCHEME_FP8_KARATSUBA}
OZ2_MODE_ACCURATE = 0
OZ2_MODE_FAST = 1
_MODES = {"accurate": OZ2_MODE_ACCURATE, "fast": OZ2_MODE_FAST}

# tuning knobs (include/oz2.h OZ2_TUNE_*): schedule only, results are bit-identical
TUNE = {
    "cta_group": 0, "sync_lead": 1, "sync_chunk": 2, "l2_promo": 3, "max_units": 4,
    "tma_hint_a": 5, "tma_hint_b": 6, "mod_split": 7, "fused_crt": 8, "sq_order": 9,
    "crt_generic": 10, "host_blocks": 11, "kcat": 12, "prescale_2read": 13,
    "epi_sleep": 14, "digits_fma": 15, "tile_n": 16,
}

_c_int64 = ctypes.c_int64
_vp = ctypes.c_void_p


class oz2_options(ctypes.Structure):
    _fields_ = [
        ("e_prime_a", _vp), ("e_prime_b", _vp), ("abar", _vp), ("bbar", _vp),
        ("rmax", _vp), ("smax", _vp), ("e_mu", _vp), ("e_nu", _vp),
        ("digits_a", _vp), ("digits_b", _vp), ("residues", _vp),
        ("e_mu_in", _vp), ("e_nu_in", _vp),
        ("timing_ms", _vp),
        ("set_mode", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("set_scheme", ctypes.c_int32), ("scheme", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 4),
    ]


class oz2_plan_info(ctypes.Structure):
    _fields_ = [
        ("num_moduli", ctypes.c_int32), ("num_planes", ctypes.c_int32),
        ("num_limbs", ctypes.c_int32), ("num_squares", ctypes.c_int32),
        ("p_prime", ctypes.c_float), ("delta", ctypes.c_float), ("f_k", ctypes.c_float),
        ("log2_P", ctypes.c_double),
        ("P_limbs", ctypes.c_uint32 * 12),
        ("w_limbs", (ctypes.c_uint32 * 12) * 33),
        ("fast_H", ctypes.c_double),
    ]


# (name, restype, argtypes) -- the full exported surface of include/oz2.h
SIGNATURES = [
    ("oz2_dgemm", ctypes.c_int,
     [ctypes.c_char, ctypes.c_char, _c_int64, _c_int64, _c_int64, ctypes.c_double, _vp, _c_int64,
      _vp, _c_int64, ctypes.c_double, _vp, _c_int64, ctypes.c_int]),
    ("oz2_dgemm_ex", ctypes.c_int,
     [ctypes.c_char, ctypes.c_char, _c_int64, _c_int64, _c_int64, ctypes.c_double, _vp, _c_int64,
      _vp, _c_int64, ctypes.c_double, _vp, _c_int64, ctypes.c_int, ctypes.POINTER(oz2_options)]),
    ("oz2_set_stream", ctypes.c_int, [_vp]),
    ("oz2_set_mode", ctypes.c_int, [ctypes.c_int]),
    ("oz2_set_scheme", ctypes.c_int, [ctypes.c_int]),
    ("oz2_get_scheme", ctypes.c_int, []),
    ("oz2_get_mode", ctypes.c_int, []),
    ("oz2_workspace_size", ctypes.c_size_t,
     [ctypes.c_char, ctypes.c_char, _c_int64, _c_int64, _c_int64, ctypes.c_int]),
    ("oz2_set_workspace", ctypes.c_int, [_vp, ctypes.c_size_t]),
    ("oz2_set_blocking", ctypes.c_int, [_c_int64, _c_int64]),
    ("oz2_get_blocking", ctypes.c_int, [ctypes.POINTER(_c_int64), ctypes.POINTER(_c_int64)]),
    ("oz2_workspace_size_blocked", ctypes.c_size_t, [_c_int64, _c_int64, _c_int64, ctypes.c_int, _c_int64, _c_int64]),
    ("oz2_plan_blocking", ctypes.c_int,
     [_c_int64, _c_int64, _c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(_c_int64), ctypes.POINTER(_c_int64)]),
    ("oz2_get_status", ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
    ("oz2_set_timing", ctypes.c_int, [ctypes.c_int]),
    ("oz2_get_timing", ctypes.c_int, [ctypes.POINTER(ctypes.c_float), ctypes.c_int]),
    ("oz2_finalize", ctypes.c_int, []),
    ("oz2_set_tuning", ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    ("oz2_get_tuning", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("oz2_reset_tuning", None, []),
    ("oz2_moduli", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int32)]),
    ("oz2_plan_query", ctypes.c_int, [ctypes.c_int, _c_int64, ctypes.POINTER(oz2_plan_info)]),
    ("oz2_version", ctypes.c_char_p, []),
    ("oz2_fp8_gemm_raw", ctypes.c_int, [_vp, _vp, _vp, _c_int64, _c_int64, _c_int64]),
    ("oz2_int8_gemm_raw", ctypes.c_int, [_vp, _vp, _vp, _c_int64, _c_int64, _c_int64]),
    ("oz2_fp8_gemm_bound", ctypes.c_int, [_vp, _vp, _vp, _vp, _c_int64, _c_int64, _c_int64]),
    ("oz2_last_cuda_error", ctypes.c_int, [ctypes.c_char_p, ctypes.c_int]),
]

_lib = None


def lib():
    """The loaded liboz2.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -m paper_2603_10634_b200._build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ch(t):
    return t.encode() if isinstance(t, str) else t


def _check(rc, what):
    if rc != OZ2_SUCCESS:
        raise RuntimeError(f"{what} failed with status {rc}")
    return rc


# ---- 1:1 wrappers of the C ABI (pointers are ints) ---------------------------------

def oz2_dgemm(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_moduli):
    return lib().oz2_dgemm(_ch(transa), _ch(transb), m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                           num_moduli)


def oz2_dgemm_ex(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, num_moduli, opt):
    return lib().oz2_dgemm_ex(_ch(transa), _ch(transb), m, n, k, alpha, A, lda, B, ldb, beta, C,
                              ldc, num_moduli, ctypes.byref(opt) if opt is not None else None)


def oz2_set_stream(stream):
    return lib().oz2_set_stream(stream)


def oz2_set_mode(mode):
    """mode: OZ2_MODE_ACCURATE / OZ2_MODE_FAST or "accurate" / "fast"."""
    return lib().oz2_set_mode(_MODES.get(mode, mode))


def oz2_get_mode():
    return lib().oz2_get_mode()


def oz2_set_scheme(scheme):
    """scheme: OZ2_SCHEME_FP8 / OZ2_SCHEME_INT8 / OZ2_SCHEME_FP8_KARATSUBA or "fp8" / "int8" /
    "karatsuba"."""
    return lib().oz2_set_scheme(_SCHEMES.get(scheme, scheme))


def oz2_get_scheme():
    return lib().oz2_get_scheme()


def oz2_workspace_size(transa, transb, m, n, k, num_moduli):
    return lib().oz2_workspace_size(_ch(transa), _ch(transb), m, n, k, num_moduli)


def oz2_set_workspace(ptr, nbytes):
    return lib().oz2_set_workspace(ptr, nbytes)


def oz2_set_blocking(mb, nb):
    return lib().oz2_set_blocking(mb, nb)


def oz2_get_blocking():
    mb, nb = _c_int64(0), _c_int64(0)
    _check(lib().oz2_get_blocking(ctypes.byref(mb), ctypes.byref(nb)), "oz2_get_blocking")
    return mb.value, nb.value


def oz2_workspace_size_blocked(m, n, k, num_moduli, mb, nb):
    return lib().oz2_workspace_size_blocked(m, n, k, num_moduli, mb, nb)


def oz2_plan_blocking(m, n, k, num_moduli, nbytes):
    """(status, mb, nb) for a workspace of nbytes (host only)."""
    mb, nb = _c_int64(0), _c_int64(0)
    rc = lib().oz2_plan_blocking(m, n, k, num_moduli, nbytes, ctypes.byref(mb), ctypes.byref(nb))
    return rc, mb.value, nb.value


def oz2_get_status():
    s = ctypes.c_int32(0)
    _check(lib().oz2_get_status(ctypes.byref(s)), "oz2_get_status")
    return s.value


def oz2_set_timing(enable):
    return lib().oz2_set_timing(1 if enable else 0)


PHASES = ["prescale", "bound_gemm", "exponents", "digits", "residue_gemm", "crt", "total"]


def oz2_get_timing():
    """Per-phase ms of the last timed call (see include/oz2.h), as a dict."""
    buf = (ctypes.c_float * 7)()
    _check(lib().oz2_get_timing(buf, 7), "oz2_get_timing")
    return dict(zip(PHASES, list(buf)))


def oz2_finalize():
    return lib().oz2_finalize()


def oz2_set_tuning(knob, value):
    """knob: OZ2_TUNE_* number or its lower-case name in TUNE."""
    return lib().oz2_set_tuning(TUNE.get(knob, knob), int(value))


def oz2_get_tuning(knob):
    v = ctypes.c_int(0)
    _check(lib().oz2_get_tuning(TUNE.get(knob, knob), ctypes.byref(v)), "oz2_get_tuning")
    return v.value


def oz2_reset_tuning():
    lib().oz2_reset_tuning()


class tuning:
    """Context manager: ``with tuning(cta_group=1, mod_split=0): ...`` sets knobs of the
    calling thread and restores the previous values on exit."""

    def __init__(self, **knobs):
        self.knobs = knobs
        self.prev = {}

    def __enter__(self):
        for k, v in self.knobs.items():
            self.prev[k] = oz2_get_tuning(k)
            _check(oz2_set_tuning(k, v), f"oz2_set_tuning({k}={v})")
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            oz2_set_tuning(k, v)
        return False


def oz2_moduli(num_moduli):
    out = (ctypes.c_int32 * num_moduli)()
    _check(lib().oz2_moduli(num_moduli, out), "oz2_moduli")
    return list(out)


def oz2_plan_query(num_moduli, k):
    info = oz2_plan_info()
    _check(lib().oz2_plan_query(num_moduli, k, ctypes.byref(info)), "oz2_plan_query")
    return info


def oz2_version():
    return lib().oz2_version().decode()


def oz2_fp8_gemm_raw(a, b, C32, m, n, k):
    return lib().oz2_fp8_gemm_raw(a, b, C32, m, n, k)


def oz2_int8_gemm_raw(a, b, C32, m, n, k):
    return lib().oz2_int8_gemm_raw(a, b, C32, m, n, k)


def oz2_last_cuda_error():
    """(code, name) of the CUDA error behind this thread's last OZ2_ERR_CUDA."""
    buf = ctypes.create_string_buffer(128)
    code = lib().oz2_last_cuda_error(buf, 128)
    return code, buf.value.decode()


def oz2_fp8_gemm_bound(a, b, rmax, smax, m, n, k):
    return lib().oz2_fp8_gemm_bound(a, b, rmax, smax, m, n, k)


# ---- torch convenience (still only marshalling) ----------------------------------

_ws = {}


def _bind_stream_and_workspace(torch, device, nbytes):
    """Point the library at torch's current stream and a torch-owned workspace.

    The library's calls are asynchronous on that stream and its state is per host thread,
    so the cached scratch buffer is keyed by (thread, device, stream): two threads, or two
    streams of one thread, never share one.  record_stream keeps the caching allocator
    from handing the buffer out again while the stream's kernels may still use it."""
    import threading
    stream = torch.cuda.current_stream(device)
    oz2_set_stream(stream.cuda_stream)
    dev = device.index if device.index is not None else torch.cuda.current_device()
    key = (threading.get_ident(), dev, stream.cuda_stream)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            buf.record_stream(stream)
        _ws[key] = None
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
        _ws[key] = buf
    buf.record_stream(stream)
    oz2_set_workspace(buf.data_ptr(), buf.numel())


def _colmajor(X):
    """(tensor, trans, ld) with op(stored) == X for a 2-D float64 CUDA tensor."""
    r, c = X.shape
    s0, s1 = X.stride()
    if s0 == 1 and s1 >= max(1, r):
        return X, "N", s1
    if s1 == 1 and s0 >= max(1, c):
        return X, "T", s0
    X = X.t().contiguous().t()
    return X, "N", X.stride(1)


def dgemm(A, B, alpha=1.0, beta=0.0, C=None, num_moduli=13, mode=None, scheme=None):
    """C <- alpha A @ B + beta C on torch float64 CUDA tensors via oz2_dgemm_ex.

    Any 2-D strided layout is accepted for A, B and C; a new C is column-major (Fortran
    order).  ``mode`` ("accurate" / "fast") and ``scheme`` ("fp8" / "int8" / "karatsuba")
    apply to this call only (oz2_options.set_mode / set_scheme); None keeps the thread's
    setting."""
    import torch
    assert A.dtype == torch.float64 and B.dtype == torch.float64
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    if C is None:
        C = torch.empty((n, m), dtype=torch.float64, device=A.device).t()
        beta = 0.0
    assert C.shape == (m, n) and C.dtype == torch.float64
    opt = oz2_options()
    if mode is not None:
        opt.set_mode, opt.mode = 1, _MODES.get(mode, mode)
    if scheme is not None:
        opt.set_scheme, opt.scheme = 1, _SCHEMES.get(scheme, scheme)
    A_, ta, lda = _colmajor(A)
    B_, tb, ldb = _colmajor(B)
    s0, s1 = C.stride()
    if s0 == 1 and s1 >= max(1, m):
        ws = oz2_workspace_size(ta, tb, m, n, k, num_moduli)
        _bind_stream_and_workspace(torch, A.device, ws)
        _check(oz2_dgemm_ex(ta, tb, m, n, k, alpha, A_.data_ptr(), lda, B_.data_ptr(), ldb, beta,
                            C.data_ptr(), s1, num_moduli, opt), "oz2_dgemm_ex")
        return C
    if s1 == 1 and s0 >= max(1, n):
        # row-major C: compute C^T = B^T A^T into the column-major view of C^T
        tb2 = "T" if tb == "N" else "N"
        ta2 = "T" if ta == "N" else "N"
        ws = oz2_workspace_size(tb2, ta2, n, m, k, num_moduli)
        _bind_stream_and_workspace(torch, A.device, ws)
        _check(oz2_dgemm_ex(tb2, ta2, n, m, k, alpha, B_.data_ptr(), ldb, A_.data_ptr(), lda, beta,
                            C.data_ptr(), s0, num_moduli, opt), "oz2_dgemm_ex")
        return C
    # any other view (e.g. C[:, ::2]): compute into a column-major temporary, copy back
    T = torch.empty((n, m), dtype=torch.float64, device=C.device).t()
    if beta != 0.0:
        T.copy_(C)
    dgemm(A, B, alpha=alpha, beta=beta, C=T, num_moduli=num_moduli, mode=mode, scheme=scheme)
    C.copy_(T)
    return C
