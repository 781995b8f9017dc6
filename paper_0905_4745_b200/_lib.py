"""ctypes binding of libminnorm_b200.so (include/minnorm_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_0905_4745_b200/csrc``).  There is no fallback: if the
library is missing, importing the solver fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MNB_LIB_PATH: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("MNB_LIB_PATH") or os.path.join(_HERE, "libminnorm_b200.so")

MNB_OK = 0
MNB_ERR_INVALID_ARGUMENT = 1
MNB_ERR_CONFIG = 2
MNB_ERR_DIMENSION = 3
MNB_ERR_RANK_DEFICIENCY = 4
MNB_ERR_CUDA = 5
MNB_ERR_NCCL = 6
MNB_ERR_UNSUPPORTED = 7
MNB_ERR_OUT_OF_MEMORY = 8
MNB_ERR_INTERNAL = 9
MNB_ERR_PARSE = 10

MNB_C128 = 0
MNB_F64 = 1
MNB_HOST = 0
MNB_DEVICE = 1
MNB_HOST_ASYNC = 2

FIELDS = {"d": 0, "zeta": 1, "zeta_tilde": 2, "theta": 3, "theta_tilde": 4, "cos_theta": 5, "sin_theta": 6,
          "cos_theta_tilde": 7, "sin_theta_tilde": 8, "perm": 9, "perm_tilde": 10, "sample": 11}


class SolverConfigC(ctypes.Structure):
    _fields_ = [("sketch_size", ctypes.c_int64), ("alpha", ctypes.c_double), ("epsilon", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("sampling", ctypes.c_int32), ("capture_c", ctypes.c_int32),
                ("lsq_max_iterations", ctypes.c_int64)]


class SolveReportC(ctypes.Structure):
    _fields_ = [("step_seconds", ctypes.c_double * 5), ("c_norm_ratio", ctypes.c_double),
                ("residual_norm", ctypes.c_double), ("lsq_iterations", ctypes.c_int64),
                ("lsq_converged", ctypes.c_int32), ("qr_path", ctypes.c_int32), ("sketch_size", ctypes.c_int64),
                ("lsq_tau", ctypes.c_double), ("lsq_achieved_excess", ctypes.c_double),
                ("param_seconds", ctypes.c_double), ("total_seconds", ctypes.c_double),
                ("sketch_seconds", ctypes.c_double * 2), ("redistribute_seconds", ctypes.c_double),
                ("qr_seconds", ctypes.c_double * 2), ("pcg_seconds", ctypes.c_double),
                ("pcg_pass_ms_sum", ctypes.c_double), ("pcg_pass_launches", ctypes.c_int64),
                ("sketch_kernel_ms", ctypes.c_double * 4), ("kernel_launches", ctypes.c_int64),
                ("world_size", ctypes.c_int64)]


class LsqConfigC(ctypes.Structure):
    _fields_ = [("sketch_size", ctypes.c_int64), ("tau", ctypes.c_double), ("max_iterations", ctypes.c_int64),
                ("stream_seed", ctypes.c_uint64), ("sampling", ctypes.c_int32), ("reserved0", ctypes.c_int32)]


class ClassicalReportC(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("refinements", ctypes.c_int32), ("residual_norm", ctypes.c_double),
                ("seconds", ctypes.c_double)]


class LsqSolutionC(ctypes.Structure):
    _fields_ = [("achieved_excess", ctypes.c_double), ("iterations", ctypes.c_int64),
                ("converged", ctypes.c_int32), ("reserved0", ctypes.c_int32)]


# every symbol include/minnorm_b200.h declares (tests check the export table)
EXPORTS = [
    "mnb_last_error", "mnb_last_deficient_columns", "mnb_version", "mnb_context_create", "mnb_nccl_unique_id",
    "mnb_context_create_distributed", "mnb_context_destroy", "mnb_context_set_stream", "mnb_shard_columns",
    "mnb_redistribute_plan", "mnb_last_parse_location", "mnb_mm_read_dims", "mnb_mm_read", "mnb_mm_write",
    "mnb_generate_instance",
    "mnb_set_matrix", "mnb_solver_config_default", "mnb_solve_randomized", "mnb_solve_classical",
    "mnb_solve_least_squares",
    "mnb_srft_build", "mnb_srft_from_fields", "mnb_srft_destroy", "mnb_srft_get_field", "mnb_srft_dims",
    "mnb_srft_apply_h", "mnb_srft_apply", "mnb_srft_apply_adjoint", "mnb_srft_apply_to_columns", "mnb_dft",
    "mnb_apply_adjoint_matrix", "mnb_bench_pcg_pass", "mnb_chol_upper", "mnb_trtri_upper", "mnb_csne_solve",
]

_lib = None


def load():
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    # libnccl.so.2 is one soname for two builds here: the system NCCL this library links and the newer
    # one torch bundles.  Whichever loads first serves both, and torch needs symbols only its own
    # build has (ncclDevCommCreate), so torch (when installed) goes first; the NCCL API this library
    # calls is in both.
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, u64, ci, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
    pvp = ctypes.POINTER(ctypes.c_void_p)
    L.mnb_last_error.restype = ctypes.c_char_p
    L.mnb_last_deficient_columns.restype = i64
    L.mnb_version.restype = ctypes.c_char_p
    L.mnb_context_create.argtypes = [ci, pvp]
    L.mnb_nccl_unique_id.argtypes = [dp]
    L.mnb_context_create_distributed.argtypes = [ci, ci, ci, dp, pvp]
    L.mnb_context_destroy.argtypes = [vp]
    L.mnb_context_destroy.restype = None
    L.mnb_context_set_stream.argtypes = [vp, vp]
    L.mnb_shard_columns.argtypes = [i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.mnb_last_parse_location.argtypes = [ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.mnb_last_parse_location.restype = None
    L.mnb_mm_read_dims.argtypes = [ctypes.c_char_p, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.mnb_mm_read.argtypes = [ctypes.c_char_p, dp, i64, i64]
    L.mnb_mm_write.argtypes = [ctypes.c_char_p, dp, i64, i64]
    L.mnb_generate_instance.argtypes = [i64, i64, ctypes.c_double, u64, dp, dp, dp]
    L.mnb_redistribute_plan.argtypes = [i64, i64, ci, ci, ctypes.POINTER(i64)]
    L.mnb_set_matrix.argtypes = [vp, ci, i64, i64, i64, i64, dp, i64, ci]
    L.mnb_solver_config_default.argtypes = [ctypes.POINTER(SolverConfigC)]
    L.mnb_solver_config_default.restype = None
    L.mnb_solve_randomized.argtypes = [vp, dp, ci, ctypes.POINTER(SolverConfigC), dp, ci, dp,
                                       ctypes.POINTER(SolveReportC)]
    L.mnb_solve_least_squares.argtypes = [vp, dp, ci, ctypes.POINTER(LsqConfigC), dp, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(LsqSolutionC)]
    L.mnb_solve_classical.argtypes = [vp, dp, ci, dp, ci, ctypes.POINTER(ClassicalReportC)]
    L.mnb_apply_adjoint_matrix.argtypes = [vp, dp, ci, dp, ci, dp]
    L.mnb_srft_build.argtypes = [i64, i64, u64, ci, pvp]
    L.mnb_srft_from_fields.argtypes = [i64, i64, ci] + [dp] * 8 + [pvp]
    L.mnb_srft_destroy.argtypes = [vp]
    L.mnb_srft_destroy.restype = None
    L.mnb_srft_get_field.argtypes = [vp, ci, dp]
    L.mnb_srft_dims.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    for f in ("mnb_srft_apply_h", "mnb_srft_apply", "mnb_srft_apply_adjoint"):
        getattr(L, f).argtypes = [vp, vp, dp, dp]
    L.mnb_srft_apply_to_columns.argtypes = [vp, vp, dp, ci]
    L.mnb_dft.argtypes = [vp, i64, dp, ci]
    L.mnb_bench_pcg_pass.argtypes = [vp, ci, ctypes.POINTER(ctypes.c_double)]
    L.mnb_chol_upper.argtypes = [vp, dp, i64, ctypes.c_double, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    L.mnb_trtri_upper.argtypes = [vp, dp, i64, dp, ctypes.POINTER(ctypes.c_double)]
    L.mnb_csne_solve.argtypes = [vp, dp, i64, i64, dp, dp, ctypes.POINTER(ctypes.c_double)]
    _lib = L
    return L


def last_error() -> str:
    return load().mnb_last_error().decode(errors="replace")
