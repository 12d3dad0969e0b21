"""ctypes binding of the C ABI in include/stg_cuda.h (libstg_cuda.so).

There is no fallback: if the in-tree CUDA library is missing or fails to
load, every entry point raises.  Build it with ``python -m
paper_2201_05800_b200.build`` (``__graft_entry__.build()`` does this).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libstg_cuda.so"

STG_OK, STG_ERR_INVALID, STG_ERR_RUNTIME, STG_ERR_NONCONVERGENCE, STG_ERR_CUDA = 0, 1, 2, 3, 4
STG_ERR_ADMISSIBILITY = 5
STG_MODEL_ADVECTION, STG_MODEL_BURGERS, STG_MODEL_ADVDIFF, STG_MODEL_EULER = 0, 1, 2, 3
STG_FIELD_CONSTANT, STG_FIELD_ROTATING = 0, 1
STG_FORM_A, STG_FORM_A_INV = 0, 1
STG_LINEAR_AUTO, STG_LINEAR_GMRES = 0, 3
STG_KERNEL_AUTO, STG_KERNEL_GENERIC, STG_KERNEL_FAST = 0, 1, 2
STG_PRECOND_NONE, STG_PRECOND_TBLOCK, STG_PRECOND_EBLOCK, STG_PRECOND_AUTO = 0, 1, 2, 3
STG_PRECOND_JACOBI = 4
STG_PRECOND_SWEEP = 5
STG_PRECOND_POLY = 6
STG_MAX_HISTORY = 64

# every symbol include/stg_cuda.h declares
EXPORTS = (
    "stg_newton_config_default", "stg_last_error", "stg_create", "stg_destroy",
    "stg_set_stream", "stg_set_kernel", "stg_sizes", "stg_constants",
    "stg_spatial_rhs", "stg_spatial_jvp", "stg_st_residual", "stg_st_jvp",
    "stg_stage_residual", "stg_stage_jvp", "stg_gmres_st", "stg_st_precond_apply",
    "stg_stdg_step", "stg_rk_step", "stg_stdg_integrate", "stg_rk_integrate",
    "stg_st_residual_host", "stg_stdg_step_host", "stg_rk_step_host", "stg_kernel_launches",
    "stg_lgl_rule", "stg_diff_matrix", "stg_lobatto_tableau",
    "stg_device_alloc", "stg_device_free", "stg_memcpy", "stg_device_synchronize",
    "stg_host_alloc", "stg_host_free",
)


class StgDesc(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int), ("degree", ctypes.c_int), ("n_tau", ctypes.c_int),
        ("model", ctypes.c_int), ("cells", ctypes.c_int * 3), ("lower", ctypes.c_double * 3),
        ("upper", ctypes.c_double * 3), ("velocity", ctypes.c_double * 3),
        ("velocity_field", ctypes.c_int), ("eps", ctypes.c_double), ("eta", ctypes.c_double),
        ("gamma", ctypes.c_double),
    ]


class StgNewtonConfig(ctypes.Structure):
    _fields_ = [
        ("abs_tol", ctypes.c_double), ("rel_tol", ctypes.c_double), ("max_iter", ctypes.c_int),
        ("linear", ctypes.c_int), ("gmres_restart", ctypes.c_int), ("gmres_tol", ctypes.c_double),
        ("gmres_max_it", ctypes.c_int), ("fd_eps", ctypes.c_double), ("precond", ctypes.c_int),
    ]


class StgSolveInfo(ctypes.Structure):
    _fields_ = [
        ("newton_iterations", ctypes.c_int), ("linear_iterations", ctypes.c_int),
        ("final_residual", ctypes.c_double), ("n_history", ctypes.c_int),
        ("residual_history", ctypes.c_double * STG_MAX_HISTORY),
        ("failed_step", ctypes.c_int),
    ]


_LIB = None
_vp = ctypes.c_void_p
_d = ctypes.c_double
_i = ctypes.c_int


def load() -> ctypes.CDLL:
    """Load libstg_cuda.so (raises if it has not been built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("STG_CUDA_LIB") or LIB_PATH)  # A/B builds (scripts/variants)
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension first "
            "(python -m paper_2201_05800_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(str(path))
    L.stg_last_error.restype = ctypes.c_char_p
    L.stg_last_error.argtypes = [_vp]
    L.stg_newton_config_default.argtypes = [ctypes.POINTER(StgNewtonConfig)]
    L.stg_newton_config_default.restype = None
    L.stg_create.argtypes = [ctypes.POINTER(StgDesc), ctypes.POINTER(_vp)]
    L.stg_destroy.argtypes = [_vp]
    L.stg_destroy.restype = None
    L.stg_set_stream.argtypes = [_vp, _vp]
    L.stg_set_kernel.argtypes = [_vp, _i]
    L.stg_sizes.argtypes = [_vp, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_longlong)]
    L.stg_constants.argtypes = [_vp, _vp, _vp, _vp]
    L.stg_kernel_launches.argtypes = [_vp]
    L.stg_kernel_launches.restype = ctypes.c_longlong
    L.stg_spatial_rhs.argtypes = [_vp, _d, _vp, _vp]
    L.stg_spatial_jvp.argtypes = [_vp, _d, _vp, _vp, _vp]
    L.stg_st_residual.argtypes = [_vp, _d, _d, _vp, _vp, _vp]
    L.stg_st_jvp.argtypes = [_vp, _d, _d, _vp, _vp, _vp, _d]
    L.stg_stage_residual.argtypes = [_vp, _i, _d, _d, _vp, _vp, _vp]
    L.stg_stage_jvp.argtypes = [_vp, _i, _d, _d, _vp, _vp, _vp, _d]
    L.stg_st_precond_apply.argtypes = [_vp, _d, _vp, _i, _vp, _vp]
    L.stg_stdg_integrate.argtypes = [_vp, _d, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp]
    L.stg_rk_integrate.argtypes = [_vp, _i, _d, _vp, _d, _i, _vp, _vp, _vp, _vp, _vp]
    L.stg_gmres_st.argtypes = [_vp, _d, _d, _vp, _vp, _vp, _i, _d, _i, _i, ctypes.POINTER(_i),
                               ctypes.POINTER(_d)]
    cfgp = ctypes.POINTER(StgNewtonConfig)
    infop = ctypes.POINTER(StgSolveInfo)
    L.stg_stdg_step.argtypes = [_vp, _d, _d, _vp, cfgp, _vp, _vp, infop]
    L.stg_rk_step.argtypes = [_vp, _i, _d, _d, _vp, cfgp, _vp, _vp, infop]
    L.stg_st_residual_host.argtypes = [_vp, _d, _d, _vp, _vp, _vp]
    L.stg_stdg_step_host.argtypes = [_vp, _d, _d, _vp, cfgp, _vp, _vp, infop]
    L.stg_rk_step_host.argtypes = [_vp, _i, _d, _d, _vp, cfgp, _vp, _vp, infop]
    L.stg_lgl_rule.argtypes = [_i, _vp, _vp]
    L.stg_diff_matrix.argtypes = [_i, _vp]
    L.stg_lobatto_tableau.argtypes = [_i, _vp, _vp, _vp]
    L.stg_device_alloc.argtypes = [ctypes.c_longlong, ctypes.POINTER(_vp)]
    L.stg_device_free.argtypes = [_vp]
    L.stg_host_alloc.argtypes = [ctypes.c_longlong, ctypes.POINTER(_vp)]
    L.stg_host_free.argtypes = [_vp]
    L.stg_memcpy.argtypes = [_vp, _vp, ctypes.c_longlong, _i]
    _LIB = L
    return L
