"""ctypes binding of libgvp_b200.so (the C ABI in include/gvp_b200.h).

This is the reference-side FFI a maintainer would add to ``gvplan``: every
function takes C-contiguous float64 numpy arrays (host memory) and maps the
library's status codes onto the reference's exception types
(INTEGRATION.md). There is no CPU fallback: if the library or a CUDA device
is missing, the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GVP_B200_LIB", os.path.join(_HERE, "libgvp_b200.so"))

GVP_OK = 0
GVP_ERR_NOT_SPD = 1
GVP_ERR_NONFINITE = 2
GVP_ERR_NO_FEASIBLE_STEP = 3
GVP_ERR_SQRT = 4
GVP_ERR_ARG = -1
GVP_ERR_UNSUPPORTED = -2
GVP_ERR_CUDA = -3
GVP_ERR_NO_DEVICE = -4
GVP_WHERE_MEAN_SOLVE_BIAS = 1 << 30
GVP_NREC = 8

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class NativeLibraryError(RuntimeError):
    """libgvp_b200.so could not be loaded or a CUDA call failed."""


class PlanConfig(C.Structure):
    """gvp_plan_config (include/gvp_b200.h)."""

    _fields_ = [("kl_bound", C.c_double), ("beta_min", C.c_double), ("beta_max", C.c_double),
                ("temp_low", C.c_double), ("temp_high", C.c_double),
                ("collision_tol", C.c_double), ("tol_mean", C.c_double),
                ("tol_cost", C.c_double), ("init_cov_scale", C.c_double),
                ("max_iters", C.c_int32), ("spec_lanes", C.c_int32)]


# name -> (restype, argtypes)
_SIGS = {
    "gvp_last_error": (C.c_char_p, []),
    "gvp_version": (C.c_char_p, []),
    "gvp_device_count": (C.c_int, []),
    "gvp_factor_expectations": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _dp, C.c_int64, _dp,
                                          C.c_int32, _i64p, _dp, C.c_double, C.c_double,
                                          C.c_double, C.c_int32, _dp, _dp, _dp, _i64p]),
    "gvp_evaluate_factors": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _dp, C.c_int64, _dp,
                                       C.c_int32, _i64p, _dp, C.c_double, C.c_double, C.c_double,
                                       _dp, _dp, _dp, _i64p, _i64p]),
    "gvp_gbp_marginals": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _dp, _i64p]),
    "gvp_gbp_mean_solve": (C.c_int, [_dp, _dp, _dp, C.c_int64, C.c_int32, _dp, _i64p]),
    "gvp_logdet_block_tridiag": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _i64p]),
    "gvp_proximal_update": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int64,
                                      C.c_int32, C.c_double, C.c_double, _dp, _dp, _dp, _i64p]),
    "gvp_select_step_size": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int64,
                                       C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                       _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int32, _i32p,
                                       _i64p]),
    "gvp_select_step_size_ld": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int64,
                                          C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                          _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int32, _i32p,
                                          _i64p, C.c_double, _dp]),
    "gvp_engine_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int64, C.c_int32,
                                    C.c_int32, _dp, C.c_int32, _i64p, _dp, C.c_double, C.c_double,
                                    C.c_double, _dp, _dp, C.c_int64, C.POINTER(PlanConfig)]),
    "gvp_engine_destroy": (None, [C.c_void_p]),
    "gvp_engine_load": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _dp]),
    "gvp_engine_load_boundary": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
    "gvp_engine_load_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "gvp_engine_step": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
    "gvp_engine_sync": (C.c_int, [C.c_void_p]),
    "gvp_engine_step_profiled": (C.c_int, [C.c_void_p, C.c_int32, _dp]),
    "gvp_engine_step_profiled_ex": (C.c_int, [C.c_void_p, C.c_int32, _dp, C.c_int32]),
    "gvp_engine_stream": (C.c_void_p, [C.c_void_p]),
    "gvp_engine_active": (C.c_int, [C.c_void_p, _i32p]),
    "gvp_engine_get_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, _dp]),
    "gvp_engine_get_summary": (C.c_int, [C.c_void_p, _i32p, _i32p, _i32p, _i32p, _i32p]),
    "gvp_engine_get_records": (C.c_int, [C.c_void_p, _dp]),
    "gvp_engine_device_state": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_void_p)] * 5),
    "gvp_engine_launches": (C.c_int64, [C.c_void_p]),
    "gvp_engine_lanes": (C.c_int32, [C.c_void_p]),
    "gvp_engine_trace_probes": (C.c_int, [C.c_void_p, C.c_int32]),
    "gvp_engine_set_map_bank": (C.c_int, [C.c_void_p, C.c_int32, _dp, _i32p]),
    "gvp_engine_raster_map_bank": (C.c_int, [C.c_void_p, C.c_int32, _i32p, _i32p, _dp, _i32p]),
    "gvp_forward_schur_chols": (C.c_int, [_dp, _dp, C.c_int64, C.c_int32, _dp, _i64p]),
    "gvp_rasterize": (C.c_int, [C.c_int32, _i64p, _dp, C.c_double, C.c_int32, _i32p, _dp, _dp]),
    "gvp_arm_factor_expectations": (C.c_int, [C.c_int64, _dp, _dp, C.c_int32, _dp, _dp, _i32p, _dp, _i64p, _dp,
                                              C.c_double, _dp, _dp, C.c_int32, _i32p, _dp, C.c_double,
                                              C.c_double, _dp, _dp, _dp, _i64p]),
    "gvp_arm_create": (C.c_int, [C.POINTER(C.c_void_p), _dp, _i64p, _dp, C.c_double, _dp, _dp, C.c_int32, _i32p,
                                 _dp, C.c_double, C.c_double, C.c_int32, _dp, _dp, _i32p]),
    "gvp_arm_destroy": (None, [C.c_void_p]),
    "gvp_arm_factor_grads": (C.c_int, [C.c_void_p, C.c_int64, _dp, _dp, _dp, _dp, _dp, _i64p, _i64p]),
    "gvp_slr_quadrotor": (C.c_int, [C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, C.c_int32, C.c_double, _dp, _dp,
                                    _dp, _i32p, _i32p]),
    "gvp_prior_assemble": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _dp, _dp, _dp, C.c_double,
                                     C.c_double, C.c_double, _dp, _dp, _dp, _dp, C.c_int32, _dp, _dp, _dp, _dp,
                                     _dp, _dp, _i32p, _i32p]),
    "gvp_engine_get_probes": (C.c_int, [C.c_void_p, _dp, _i32p]),
    "gvp_prior_assemble_reg": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, _dp, _dp, _dp, C.c_double,
                                         C.c_double, C.c_double, _dp, _dp, _dp, _dp, C.c_int32, C.c_double, _dp,
                                         _dp, _dp, _dp, _dp, _dp, _i32p, _i32p]),
    "gvp_engine_step_beta": (C.c_int, [C.c_void_p, _dp]),
    "gvp_engine_get_oob": (C.c_int, [C.c_void_p, _i64p]),
    "gvp_engine_get_packed": (C.c_int, [C.c_void_p, _dp, _dp]),
    "gvp_engine_set_state": (C.c_int, [C.c_void_p, C.c_int32, _i32p, _dp, _dp, _dp]),
    "gvp_set_step_lanes": (C.c_int, [C.c_int32]),
    "gvp_chain_scratch_doubles": (C.c_int64, [C.c_int32, C.c_int64, C.c_int32, C.c_int32]),
    "gvp_gbp_marginals_dev": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p]),
}

_lib = None


def load():
    """Load the library (once) and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); the CUDA path has "
            "no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS)


def last_error() -> str:
    return load().gvp_last_error().decode()


def f64(a) -> np.ndarray:
    """C-contiguous float64 view/copy of a."""
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def ptr(a: np.ndarray):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.int64:
        return a.ctypes.data_as(_i64p)
    if a.dtype == np.int32:
        return a.ctypes.data_as(_i32p)
    raise TypeError(a.dtype)


def check(code: int, what: str):
    """Raise for infrastructure errors; numeric statuses are mapped by the
    callers (they know which reference exception applies)."""
    if code in (GVP_ERR_CUDA, GVP_ERR_NO_DEVICE):
        raise NativeLibraryError(f"{what}: {last_error()}")
    if code == GVP_ERR_ARG:
        raise ValueError(f"{what}: {last_error()}")
    if code == GVP_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {last_error()}")
    return code
