"""ctypes mirror of the POD types in include/epicorr_b200.h.

Pure type declarations (no library loading) so that both the product loader
(`_lib.py`) and the test-side oracle loader can share them.
"""
from __future__ import annotations

import ctypes as C

EPC_OK = 0
EPC_ERR_INVALID_ARGUMENT = 1
EPC_ERR_RUNTIME = 2
EPC_ERR_DOMAIN = 3
EPC_ERR_CUDA = 4
EPC_ERR_UNSUPPORTED = 5

EPC_MEM_HOST = 0
EPC_MEM_DEVICE = 1

STOP_CONVERGED, STOP_MAX_ITERATIONS, STOP_LINE_SEARCH_FAILURE, STOP_ERROR = 0, 1, 2, 3
STOP_NAMES = {0: "converged", 1: "max_iterations", 2: "line_search_failure", 3: "error"}
RHO_FIXED, RHO_ADAPTIVE, RHO_ADAPTIVE_BOUNDED = 0, 1, 2
PRECOND_NONE, PRECOND_JACOBI, PRECOND_BLOCK_JACOBI, PRECOND_SGS = 0, 1, 2, 3

dptr = C.POINTER(C.c_double)
iptr = C.POINTER(C.c_int)


class Grid(C.Structure):
    """GridSpec (proj/include/epicorr/grid.hpp:16-52)."""

    _fields_ = [("dim", C.c_int), ("m", C.c_int * 3), ("h", C.c_double * 3),
                ("origin", C.c_double * 3)]

    @classmethod
    def make(cls, m1, m2, m3=1, h=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), dim=None):
        g = cls()
        g.dim = dim if dim is not None else (2 if m3 == 1 else 3)
        g.m[:] = [m1, m2, m3]
        g.h[:] = list(h)
        g.origin[:] = list(origin)
        return g

    @property
    def n1(self):
        return self.m[0] + 1

    @property
    def faces(self):
        return (self.m[0] + 1) * self.m[1] * self.m[2]

    @property
    def cells(self):
        return self.m[0] * self.m[1] * self.m[2]

    @property
    def columns(self):
        return self.m[1] * self.m[2]

    def dims(self):
        return tuple(self.m)


class ObjectiveParams(C.Structure):
    """ObjectiveParams (proj/include/epicorr/objective.hpp:25-34)."""

    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("gamma", C.c_double),
                ("enforce_linf_box", C.c_int)]

    def __init__(self, alpha=50.0, beta=10.0, gamma=1e-3, enforce_linf_box=0):
        super().__init__(alpha, beta, gamma, int(enforce_linf_box))


class AdmmConfig(C.Structure):
    """ADMMConfig (proj/include/epicorr/admm.hpp:36-50), reference defaults."""

    _fields_ = [("rho0", C.c_double), ("rho_min", C.c_double), ("schedule", C.c_int),
                ("eps_abs", C.c_double), ("eps_rel", C.c_double), ("max_iter", C.c_int),
                ("tau_incr", C.c_double), ("tau_decr", C.c_double), ("mu", C.c_double),
                ("sqp_max_iter", C.c_int), ("sqp_tol_rel", C.c_double),
                ("check_kkt", C.c_int), ("threads", C.c_int)]

    def __init__(self, **kw):
        d = dict(rho0=1e6, rho_min=1e2, schedule=RHO_ADAPTIVE_BOUNDED, eps_abs=0.2,
                 eps_rel=0.2, max_iter=50, tau_incr=2.0, tau_decr=2.0, mu=10.0,
                 sqp_max_iter=20, sqp_tol_rel=1e-2, check_kkt=1, threads=1)
        d.update(kw)
        super().__init__(**d)


class GnConfig(C.Structure):
    """GNConfig (proj/include/epicorr/gn_pcg.hpp:26-40), reference defaults."""

    _fields_ = [("eta", C.c_double), ("max_outer", C.c_int), ("eps_obj", C.c_double),
                ("eps_iter", C.c_double), ("eps_grad", C.c_double), ("wolfe_c1", C.c_double),
                ("wolfe_c2", C.c_double), ("max_pcg", C.c_int), ("max_ls", C.c_int),
                ("precond", C.c_int), ("threads", C.c_int)]

    def __init__(self, **kw):
        d = dict(eta=0.1, max_outer=10, eps_obj=1e-3, eps_iter=1e-2, eps_grad=1e-2,
                 wolfe_c1=1e-4, wolfe_c2=0.9, max_pcg=100, max_ls=30,
                 precond=PRECOND_BLOCK_JACOBI, threads=1)
        d.update(kw)
        super().__init__(**d)


class AdmmRow(C.Structure):
    """AdmmIterRow (proj/include/epicorr/report.hpp:28-40)."""

    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("primal_res", C.c_double),
                ("dual_res", C.c_double), ("eps_pri", C.c_double), ("eps_dual", C.c_double),
                ("rho", C.c_double), ("lagrangian", C.c_double), ("kkt_violation", C.c_double),
                ("b_update_s", C.c_double), ("wall_s", C.c_double)]


class GnRow(C.Structure):
    """GnIterRow (proj/include/epicorr/report.hpp:16-26)."""

    _fields_ = [("level", C.c_int), ("iter", C.c_int), ("j_value", C.c_double),
                ("grad_norm", C.c_double), ("step", C.c_double), ("pcg_iters", C.c_int),
                ("pcg_relres", C.c_double), ("pcg_relres_prec", C.c_double),
                ("wall_s", C.c_double)]


SOLVER_GN, SOLVER_ADMM = 0, 1
RESTART_PROLONG_ALL, RESTART_B_FOR_BOTH, RESTART_AVERAGE = 1, 2, 3


class MultilevelStatus(C.Structure):
    """epc_multilevel_status: SolveReport of a multilevel solve."""

    _fields_ = [("stop", C.c_int), ("n_admm_rows", C.c_int), ("n_gn_rows", C.c_int),
                ("b_level", C.c_int), ("message", C.c_char * 256)]


class BUpdateStats(C.Structure):
    _fields_ = [("sqp_iters", C.c_long), ("qp_iters", C.c_long), ("kkt_violation", C.c_double),
                ("max_active", C.c_int)]


class SolveStatus(C.Structure):
    _fields_ = [("stop", C.c_int), ("nrows", C.c_int), ("message", C.c_char * 256)]


class ObjectiveEval(C.Structure):
    _fields_ = [("value", C.c_double), ("dist", C.c_double), ("smooth", C.c_double),
                ("pen", C.c_double), ("feasible", C.c_int)]


class PcgResult(C.Structure):
    _fields_ = [("iters", C.c_int), ("relres", C.c_double), ("relres_prec", C.c_double),
                ("reached_tol", C.c_int)]


class DualResult(C.Structure):
    _fields_ = [("primal_res", C.c_double), ("dual_res", C.c_double), ("eps_pri", C.c_double),
                ("eps_dual", C.c_double)]


def rows_to_dicts(rows, n):
    out = []
    for i in range(n):
        r = rows[i]
        out.append({name: getattr(r, name) for name, _ in r._fields_})
    return out
