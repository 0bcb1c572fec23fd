"""B200-native FP8 Ozaki-II DGEMM emulation (arxiv 2603.10634).

The compute path is liboz2.so (hand-written CUDA for sm_100a, C ABI in
include/oz2.h); this package is its Python binding plus the row-sharded
multi-GPU driver (``dist``).
"""
from .oz2 import (  # noqa: F401
    LIB_PATH, OZ2_ERR_ALLOC, OZ2_ERR_CUDA, OZ2_ERR_NONFINITE, OZ2_ERR_NOT_SUPPORTED,
    OZ2_ERR_WORKSPACE, OZ2_MODE_ACCURATE, OZ2_MODE_FAST, OZ2_SCHEME_FP8, OZ2_SCHEME_INT8, OZ2_SCHEME_FP8_KARATSUBA, OZ2_SUCCESS, SIGNATURES, dgemm, lib, oz2_dgemm, oz2_dgemm_ex,
    oz2_finalize, oz2_fp8_gemm_raw, oz2_get_status, oz2_get_timing, oz2_set_timing, PHASES, oz2_moduli, oz2_options, oz2_plan_info,
    oz2_plan_query, oz2_get_mode, oz2_set_mode, oz2_get_scheme, oz2_set_scheme, oz2_int8_gemm_raw, oz2_fp8_gemm_bound, oz2_last_cuda_error, oz2_set_stream, oz2_set_workspace, oz2_set_blocking, oz2_get_blocking,
    oz2_workspace_size_blocked, oz2_plan_blocking, oz2_version, oz2_workspace_size,
    TUNE, oz2_set_tuning, oz2_get_tuning, oz2_reset_tuning, tuning,
)
