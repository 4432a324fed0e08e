"""Loader for libepicorr_b200.so (the product). No fallback: if the CUDA
library cannot be built or loaded, every call raises."""
from __future__ import annotations

import ctypes as C
import os
import threading

from .abi import (AdmmConfig, AdmmRow, BUpdateStats, DualResult, GnConfig, GnRow, Grid,
                  MultilevelStatus,
                  ObjectiveEval, ObjectiveParams, PcgResult, SolveStatus, dptr, iptr)

HERE = os.path.dirname(os.path.abspath(__file__))
# EPC_LIB: load another build of the same sources (A/B experiments, scripts/)
LIB_PATH = os.environ.get("EPC_LIB") or os.path.join(HERE, "libepicorr_b200.so")
_lock = threading.Lock()
_lib = None

# every symbol include/epicorr_b200.h declares
EXPORTS = [
    "epc_default_params", "epc_default_admm_config", "epc_default_gn_config",
    "epc_context_create", "epc_context_destroy", "epc_set_stream", "epc_last_error",
    "epc_set_mode", "epc_profile_enable", "epc_profile_read", "epc_profile_reset",
    "epc_launch_count", "epc_reset_launch_count", "epc_admm_solve", "epc_admm_solve_batch",
    "epc_admm_solve_f32",
    "epc_b_update", "epc_z_update", "epc_dct_solve", "epc_dual_update",
    "epc_augmented_lagrangian", "epc_rho_schedule", "epc_qp_active_set_batch", "epc_gn_solve",
    "epc_objective_gn", "epc_gn_hessian_build", "epc_gn_hessian_apply", "epc_precond_apply",
    "epc_pcg", "epc_residual", "epc_build_info", "epc_bstep_timing", "epc_bstep_counters",
    "epc_slab_bstep", "epc_slab_zforward", "epc_slab_zsolve3", "epc_slab_zbackward",
    "epc_slab_zdiff", "epc_slab_scale", "epc_gnslab_objective", "epc_gnslab_hessian",
    "epc_gnslab_hv", "epc_gnslab_update", "epc_gnslab_axpy", "epc_gnslab_negate",
    "epc_gnslab_dot", "epc_default_schedule", "epc_restrict_image", "epc_prolong_field",
    "epc_multilevel_solve", "epc_avg_x1", "epc_diff_x1", "epc_diff_x1_adjoint",
    "epc_smoother_hessian_apply", "epc_tridiag_apply", "epc_tridiag_solve_batched", "epc_dct_apply",
    "epc_distance_hessian_apply", "epc_is_strictly_feasible", "epc_correct_pair", "epc_ssd", "epc_ncc", "epc_simulate_pair", "epc_write_volume", "epc_read_volume",
    "epc_permute_to_axis1", "epc_unpermute_field", "epc_admm_counters", "epc_slab_seq_sums", "epc_slab_d1_norm_inf", "epc_gn_stencil_apply", "epc_gn_cross_diag_add",
    "epc_jacobi_apply", "epc_admm_solve_batch_devices", "epc_nccl_unique_id", "epc_nccl_comm_create",
    "epc_nccl_comm_destroy", "epc_slab_admm_solve", "epc_guard_check",
]


class _Tolerant:
    """Declares argtypes only for symbols present (the ABI test checks that
    all of EXPORTS are)."""

    def __init__(self, lib):
        self.__dict__["_l"] = lib

    def __getattr__(self, name):
        try:
            return getattr(self._l, name)
        except AttributeError:
            return C.CFUNCTYPE(None)()  # dummy sink for argtypes


def _declare(L):
    L = _Tolerant(L)
    G, P = C.POINTER(Grid), C.POINTER(ObjectiveParams)
    A, N = C.POINTER(AdmmConfig), C.POINTER(GnConfig)
    X = C.c_void_p
    L.epc_context_create.argtypes = [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]
    L.epc_context_destroy.argtypes = [X]
    L.epc_context_destroy.restype = None
    L.epc_set_stream.argtypes = [X, C.c_void_p]
    L.epc_last_error.argtypes = [X]
    L.epc_last_error.restype = C.c_char_p
    L.epc_set_mode.argtypes = [X, C.c_int]
    L.epc_admm_counters.argtypes = [X, C.POINTER(C.c_longlong)]
    L.epc_slab_seq_sums.argtypes = [X, C.c_longlong, X, X, X, X, dptr]
    L.epc_slab_d1_norm_inf.argtypes = [X, G, C.c_int, C.c_int, X, dptr]
    L.epc_gn_stencil_apply.argtypes = [X, G, C.c_int, X, X, C.c_double, C.c_double, X, X]
    L.epc_gn_cross_diag_add.argtypes = [X, G, C.c_int, X, C.c_double, C.c_double, X]
    L.epc_jacobi_apply.argtypes = [X, C.c_longlong, C.c_int, X, X, X]
    L.epc_admm_solve_batch_devices.argtypes = [C.POINTER(C.c_void_p), C.c_int, G, C.c_int, X, X, X, X,
                                               X, X, X, X, dptr, P, A, C.c_int, C.POINTER(AdmmRow),
                                               C.c_int, C.POINTER(SolveStatus)]
    L.epc_nccl_unique_id.argtypes = [C.c_char_p]
    L.epc_guard_check.argtypes = [X, C.POINTER(C.c_int)]
    L.epc_nccl_comm_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_void_p)]
    L.epc_nccl_comm_destroy.argtypes = [X]
    L.epc_slab_admm_solve.argtypes = [X, X, C.c_int, C.c_int, G, X, X, X, X, X, X, X, X, dptr, P, A,
                                      C.c_int, C.POINTER(AdmmRow), C.c_int, C.POINTER(SolveStatus)]
    L.epc_profile_enable.argtypes = [X, C.c_int]
    L.epc_profile_read.argtypes = [X, C.POINTER(C.c_char_p), dptr, C.POINTER(C.c_long), C.c_int,
                                   C.POINTER(C.c_int)]
    L.epc_profile_reset.argtypes = [X]
    L.epc_profile_reset.restype = None
    L.epc_launch_count.argtypes = [X]
    L.epc_launch_count.restype = C.c_long
    L.epc_reset_launch_count.argtypes = [X]
    L.epc_reset_launch_count.restype = None
    L.epc_admm_solve.argtypes = [X, G, C.c_int, X, X, X, X, X, X, X, X, dptr, P, A, C.c_int,
                                 C.POINTER(AdmmRow), C.c_int, C.POINTER(SolveStatus)]
    L.epc_admm_solve_f32.argtypes = [X, G, C.c_int, X, X, X, X, X, X, X, X, dptr, P, A, C.c_int,
                                     X, C.c_int, X]
    L.epc_admm_solve_batch.argtypes = [X, G, C.c_int, C.c_int, X, X, X, X, X, X, X, X, dptr, P, A,
                                       C.c_int, C.POINTER(AdmmRow), C.c_int, C.POINTER(SolveStatus)]
    L.epc_b_update.argtypes = [X, G, C.c_int, X, X, X, X, X, C.c_double, P, A, X,
                               C.POINTER(BUpdateStats)]
    L.epc_z_update.argtypes = [X, G, C.c_int, X, X, C.c_double, C.c_double, X]
    L.epc_dct_solve.argtypes = [X, G, C.c_int, X, C.c_double, C.c_double, X]
    L.epc_dual_update.argtypes = [X, G, C.c_int, X, X, X, X, C.c_double, C.c_double, C.c_double, X,
                                  C.POINTER(DualResult)]
    L.epc_augmented_lagrangian.argtypes = [X, G, C.c_int, X, X, X, X, X, C.c_double, C.c_double, dptr]
    L.epc_rho_schedule.argtypes = [C.c_int] + [C.c_double] * 7
    L.epc_rho_schedule.restype = C.c_double
    L.epc_qp_active_set_batch.argtypes = [X, C.c_int, C.c_int, C.c_double, X, X, X, X, C.c_int, X,
                                          X, X, X, X, X]
    L.epc_gn_solve.argtypes = [X, G, C.c_int, X, X, X, X, P, N, C.c_int, C.POINTER(GnRow), C.c_int,
                               C.POINTER(SolveStatus)]
    L.epc_objective_gn.argtypes = [X, G, C.c_int, X, X, X, P, C.c_int, C.POINTER(ObjectiveEval), X, X]
    L.epc_gn_hessian_build.argtypes = [X, G, C.c_int, X, X, X, P, X, X, X]
    L.epc_gn_hessian_apply.argtypes = [X, G, C.c_int, X, X, X, P, X, X]
    L.epc_precond_apply.argtypes = [X, G, C.c_int, X, X, X, P, C.c_int, X, X]
    L.epc_pcg.argtypes = [X, G, C.c_int, X, X, X, P, C.c_int, X, C.c_double, C.c_int, X,
                          C.POINTER(PcgResult)]
    L.epc_residual.argtypes = [X, G, C.c_int, X, X, X, X]
    L.epc_build_info.restype = C.c_char_p
    L.epc_bstep_timing.argtypes = [X, C.POINTER(C.c_longlong)]
    L.epc_bstep_counters.argtypes = [X, C.POINTER(C.c_longlong)]
    D, LL, I = C.POINTER(C.c_double), C.POINTER(C.c_longlong), C.c_int
    L.epc_slab_bstep.argtypes = [X, G, I, I, X, X, X, X, X, C.c_double, P, A, X, D, LL]
    L.epc_slab_zforward.argtypes = [X, G, I, I, I, X, X, C.c_double, X]
    L.epc_slab_zsolve3.argtypes = [X, G, I, X, C.c_double, C.c_double, X]
    L.epc_slab_zbackward.argtypes = [X, G, I, I, I, X, X, X, X, C.c_double, X, X, D]
    L.epc_slab_zdiff.argtypes = [X, G, I, I, X, X, D]
    L.epc_slab_scale.argtypes = [X, C.c_longlong, X, C.c_double]
    L.epc_gnslab_objective.argtypes = [X, G, I, I, I, I, X, X, X, P, I, X, X, I, D]
    L.epc_gnslab_hessian.argtypes = [X, G, I, I, I, I, X, X, X, P, I, LL]
    L.epc_gnslab_hv.argtypes = [X, G, I, I, I, I, P, X, X, D]
    L.epc_gnslab_update.argtypes = [X, G, I, I, I, I, P, I, C.c_double, I, X, X, X, X, X, D]
    L.epc_gnslab_axpy.argtypes = [X, C.c_longlong, X, C.c_double, X, X]
    L.epc_gnslab_negate.argtypes = [X, C.c_longlong, X, X, D]
    L.epc_gnslab_dot.argtypes = [X, C.c_longlong, X, X, D]
    GA = C.POINTER(Grid)
    IPT = C.POINTER(C.c_int)
    L.epc_default_schedule.argtypes = [G, I, I, GA, I, IPT]
    L.epc_restrict_image.argtypes = [X, G, G, I, X, X]
    L.epc_prolong_field.argtypes = [X, G, G, I, X, X]
    for nm in ("epc_avg_x1", "epc_diff_x1", "epc_diff_x1_adjoint", "epc_smoother_hessian_apply"):
        getattr(L, nm).argtypes = [X, G, I, X, X]
    L.epc_tridiag_apply.argtypes = [X, G, I, X, X, X, C.c_double, X]
    L.epc_tridiag_solve_batched.argtypes = [X, G, I, X, X, X, X]
    L.epc_dct_apply.argtypes = [X, G, I, X, C.c_double, C.c_double, X]
    L.epc_distance_hessian_apply.argtypes = [X, G, I, X, X, X, X, X]
    L.epc_is_strictly_feasible.argtypes = [X, G, I, X, IPT]
    L.epc_correct_pair.argtypes = [X, G, I, X, X, X, X, X]
    L.epc_ssd.argtypes = [X, G, I, X, X, D]
    L.epc_ncc.argtypes = [X, G, I, X, X, D]
    L.epc_simulate_pair.argtypes = [X, G, I, X, X, C.c_double, C.c_ulonglong, C.c_double, X, X]
    L.epc_write_volume.argtypes = [C.c_char_p, G, I, X]
    L.epc_read_volume.argtypes = [C.c_char_p, G, IPT, X, C.c_longlong, LL]
    L.epc_permute_to_axis1.argtypes = [X, G, I, I, X, X, G]
    L.epc_unpermute_field.argtypes = [X, G, I, I, X, X, G, IPT]
    L.epc_multilevel_solve.argtypes = [X, G, I, X, X, GA, I, IPT, IPT, I, P, N, A, I, X,
                                       C.POINTER(AdmmRow), I, C.POINTER(GnRow), I,
                                       C.POINTER(MultilevelStatus)]


def load(build_if_missing=True):
    """Load (building in-tree first if missing or stale) the CUDA library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing:
            from . import build as _build
            try:
                _build.build()
            except Exception:
                if not os.path.exists(LIB_PATH):
                    raise
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libepicorr_b200.so not found at {LIB_PATH}; run build()")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
        return L
