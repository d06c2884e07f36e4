"""ctypes binding of the C ABI in include/fracprec_b200.h.

The shared library is built in-tree (``python -m paper_2112_12397_b200.build`` or
``__graft_entry__.build()``) into ``paper_2112_12397_b200/_lib/``.  There is no
fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
# FRACPREC_B200_LIB overrides the in-tree library (A/B builds of kernel variants)
LIB_PATH = os.environ.get("FRACPREC_B200_LIB") or os.path.join(_HERE, "_lib", "libfracprec_b200.so")

FP_OK, FP_INVALID_ARGUMENT, FP_NUMERICAL_ERROR, FP_CUDA_ERROR, FP_INTERNAL_ERROR = 0, 1, 2, 3, 4
FP_MEM_HOST, FP_MEM_DEVICE = 0, 1
FP_TPU, FP_TUP, FP_TUP_STAR = 0, 1, 2
FP_SMOOTHER_JACOBI, FP_SMOOTHER_SGS, FP_SMOOTHER_CHEBYSHEV, FP_SMOOTHER_MCGS = 0, 1, 2, 3


class NumericalError(RuntimeError):
    """fracprec::numerical_error (errors.hpp:15-18)."""


class CudaError(RuntimeError):
    """A CUDA failure inside the native library."""


# fp_csr / fp_block_system / the generator's spec structs: shared with the workload binding
# (workload/, a sibling of this package; its library is a dependency of this one)
if os.path.dirname(_HERE) not in sys.path:
    sys.path.insert(0, os.path.dirname(_HERE))
from workload.gen import FpBlockSystem, FpCsr, FpFractureSpec, FpWorkloadSpec  # noqa: E402,F401


class FpAmgConfig(C.Structure):
    _fields_ = [("strength_threshold", C.c_double), ("max_coarse", C.c_int32), ("pre_sweeps", C.c_int32),
                ("post_sweeps", C.c_int32), ("smoother", C.c_int32), ("prolongation_smoothing", C.c_int32),
                ("cycles_per_apply", C.c_int32), ("jacobi_omega", C.c_double), ("stall_ratio", C.c_double),
                ("max_levels", C.c_int32), ("chebyshev_degree", C.c_int32), ("chebyshev_ratio", C.c_double),
                ("power_iterations", C.c_int32), ("row_sum", C.c_int32)]


class FpPrecondConfig(C.Structure):
    _fields_ = [("variant", C.c_int32), ("amg", FpAmgConfig), ("factor_solve", C.c_int32)]


class FpGmresOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int32), ("max_iter", C.c_int32), ("scaled", C.c_int32),
                ("orthogonalization", C.c_int32), ("probe", C.c_int32)]


class FpSolveStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("restarts", C.c_int32), ("precond_applies", C.c_int32), ("final_rel_residual", C.c_double),
                ("device_seconds", C.c_double), ("kernel_launches", C.c_int64),
                ("residual_history", C.POINTER(C.c_double)),
                ("history_capacity", C.c_int32), ("history_len", C.c_int32), ("probe_ms", C.c_double),
                ("probe_launches", C.c_int32), ("reorth_steps", C.c_int32)]


class FpProfile(C.Structure):
    _fields_ = [("apply_ms", C.c_double), ("apply_bytes", C.c_double), ("apply_launches", C.c_int32),
                ("japply_ms", C.c_double), ("japply_bytes", C.c_double), ("fine_resid_ms", C.c_double),
                ("fine_resid_bytes", C.c_double), ("fine_post_ms", C.c_double), ("fine_post_bytes", C.c_double),
                ("band_ms", C.c_double), ("band_bytes", C.c_double), ("coarse_ms", C.c_double),
                ("n_levels", C.c_int32), ("level_rows", C.c_int32 * 32), ("level_nnz", C.c_int64 * 32),
                ("vcycle_ms", C.c_double * 32), ("apply_wasted_bytes", C.c_double)]


class FpAmgLevelDesc(C.Structure):
    _fields_ = [("A", FpCsr), ("P", FpCsr), ("smoother_diag", C.POINTER(C.c_double))]


class FpPrecondDesc(C.Structure):
    _fields_ = [("variant", C.c_int32), ("h_blocks", C.POINTER(C.c_double)), ("factor_matrix", FpCsr),
                ("n_levels", C.c_int32), ("levels", C.POINTER(FpAmgLevelDesc)), ("amg", FpAmgConfig),
                ("factor_solve", C.c_int32)]


# Every symbol include/fracprec_b200.h declares, with its ctypes signature (restype, argtypes).
# (include/fracprec_workload.h: libfp_workload.so, workload/gen.py SIGNATURES)
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_DP = C.POINTER(C.c_double)
SIGNATURES = {
    "fp_last_error": (C.c_char_p, []),
    "fp_version": (C.c_char_p, []),
    "fp_amg_config_default": (None, [C.POINTER(FpAmgConfig)]),
    "fp_system_create": (C.c_int, [C.POINTER(FpBlockSystem), _PP]),
    "fp_system_destroy": (None, [_P]),
    "fp_system_dims": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fp_system_apply": (C.c_int, [_P, _P, _P, C.c_int32]),
    "fp_block_scaling": (C.c_int, [_P, _DP, _DP]),
    "fp_host_precond_build": (C.c_int, [C.POINTER(FpBlockSystem), C.POINTER(FpPrecondConfig), _DP, C.c_int32, _PP]),
    "fp_host_precond_destroy": (None, [_P]),
    "fp_host_precond_levels": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fp_host_precond_matrix": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32), _DP]),
    "fp_host_precond_vector": (C.c_int, [_P, C.c_int32, C.c_int32, _DP, C.POINTER(C.c_int64)]),
    "fp_host_precond_set_upload": (C.c_int, [_P, C.c_int32, C.c_int32]),
    "fp_precond_create": (C.c_int, [_P, _P, _PP]),
    "fp_precond_upload": (C.c_int, [_P, C.POINTER(FpPrecondDesc), _PP]),
    "fp_precond_destroy": (None, [_P]),
    "fp_precond_apply": (C.c_int, [_P, _P, _P, C.c_int32]),
    "fp_amg_apply": (C.c_int, [_P, _P, _P, C.c_int32]),
    "fp_precond_inner_calls": (C.c_int64, [_P, C.c_int32]),
    "fp_precond_factor_solve": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "fp_precond_traffic": (C.c_int, [_P, _DP, C.POINTER(C.c_int32), _DP]),
    "fp_precond_profile": (C.c_int, [_P, C.c_int32, C.POINTER(FpProfile)]),
    "fp_gmres": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(FpGmresOptions), C.POINTER(FpSolveStats)]),
    "fp_workload_host_precond_build": (C.c_int, [_P, C.POINTER(FpPrecondConfig), _PP]),
    "fp_setup_backend": (C.c_int, [C.POINTER(C.c_int32)]),
    "fp_fracture_assembly_create": (C.c_int, [_P, _PP]),
    "fp_fracture_assembly_destroy": (None, [_P]),
    "fp_fracture_assembly_run": (C.c_int, [_P, _P, _P]),
    "fp_fracture_assembly_matrix": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                              C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32), _DP]),
    "fp_set_setup_backend": (C.c_int, [C.c_int32]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"fracprec_b200 native library not found at {LIB_PATH}; build it with "
            "`python -m paper_2112_12397_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    """Raise the Python image of the reference's exception classes."""
    if status == FP_OK:
        return
    msg = (lib.fp_last_error() or b"").decode()
    if status == FP_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == FP_NUMERICAL_ERROR:
        raise NumericalError(msg)
    if status == FP_CUDA_ERROR:
        raise CudaError(msg)
    raise RuntimeError(msg)
