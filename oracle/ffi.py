"""TEST INFRASTRUCTURE ONLY: ctypes front-end for the two CPU checkers.

    load("ref")     oracle/_ref/libepicorr_ref.so      (the reference library)
    load("oracle")  oracle/_build/libepicorr_oracle.so (the C restatement)

Both export oracle_api.h. Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

from paper_1607_00531_b200 import abi
from paper_1607_00531_b200.abi import (AdmmConfig, AdmmRow, BUpdateStats, DualResult, GnConfig,
                                       GnRow, Grid, ObjectiveEval, ObjectiveParams, PcgResult,
                                       SolveStatus, dptr, iptr)

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "ref": os.path.join(HERE, "_ref", "libepicorr_ref.so"),
    "oracle": os.path.join(HERE, "_build", "libepicorr_oracle.so"),
}
REFERENCE_SRC = "/root/reference/proj"
_lock = threading.Lock()
_libs = {}


def build(kind="oracle", quiet=True):
    """Compile the checker (make oracle / make ref) if it is missing."""
    target = {"oracle": "oracle", "ref": "ref"}[kind]
    if kind == "ref" and not os.path.isdir(REFERENCE_SRC):
        return False
    r = subprocess.run(["make", "-C", HERE, "-j8", target], capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build ({kind}) failed:\n{r.stdout}\n{r.stderr}")
    return True


def available(kind):
    return os.path.exists(PATHS[kind]) or (kind == "ref" and os.path.isdir(REFERENCE_SRC))


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need contiguous float64"
    return a.ctypes.data_as(dptr)


def _ip(a):
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(iptr)


class Checker:
    """One loaded checker library with numpy-level helpers."""

    def __init__(self, kind):
        self.kind = kind
        path = PATHS[kind]
        if not os.path.exists(path):
            build(kind)
        self.lib = L = C.CDLL(path)
        G, P, A, N = C.POINTER(Grid), C.POINTER(ObjectiveParams), C.POINTER(AdmmConfig), C.POINTER(GnConfig)
        L.oracle_admm_solve.argtypes = [G, dptr, dptr, dptr, dptr, dptr, dptr, dptr, dptr, dptr, P, A,
                                        C.c_int, C.POINTER(AdmmRow), C.c_int, C.POINTER(SolveStatus)]
        L.oracle_gn_solve.argtypes = [G, dptr, dptr, dptr, dptr, P, N, C.c_int, C.POINTER(GnRow),
                                      C.c_int, C.POINTER(SolveStatus)]
        L.oracle_b_update.argtypes = [G, dptr, dptr, dptr, dptr, dptr, C.c_double, P, A, dptr,
                                      C.POINTER(BUpdateStats), C.c_char_p, C.c_size_t]
        L.oracle_z_update.argtypes = [G, dptr, dptr, C.c_double, C.c_double, dptr, C.c_char_p, C.c_size_t]
        L.oracle_dct_solve.argtypes = [G, dptr, C.c_double, C.c_double, dptr, C.c_char_p, C.c_size_t]
        L.oracle_dual_update.argtypes = [G, dptr, dptr, dptr, dptr, C.c_double, C.c_double, C.c_double,
                                         dptr, C.POINTER(DualResult)]
        L.oracle_augmented_lagrangian.argtypes = [G, dptr, dptr, dptr, dptr, dptr, C.c_double, C.c_double]
        L.oracle_augmented_lagrangian.restype = C.c_double
        L.oracle_qp_active_set.argtypes = [C.c_int, C.c_double, dptr, dptr, dptr, dptr, C.c_int, dptr,
                                           dptr, iptr, iptr, C.c_char_p, C.c_size_t]
        L.oracle_verify_qp_kkt.argtypes = [C.c_int, C.c_double, dptr, dptr, dptr, dptr, dptr, iptr]
        L.oracle_verify_qp_kkt.restype = C.c_double
        L.oracle_objective_gn.argtypes = [G, dptr, dptr, dptr, P, C.c_int, C.POINTER(ObjectiveEval),
                                          dptr, dptr]
        L.oracle_gn_hessian_build.argtypes = [G, dptr, dptr, dptr, P, dptr, dptr, dptr, C.c_char_p,
                                              C.c_size_t]
        L.oracle_gn_hessian_apply.argtypes = [G, dptr, dptr, dptr, P, dptr, dptr, C.c_char_p, C.c_size_t]
        L.oracle_precond_apply.argtypes = [G, dptr, dptr, dptr, P, C.c_int, dptr, dptr, C.c_char_p,
                                           C.c_size_t]
        L.oracle_pcg.argtypes = [G, dptr, dptr, dptr, P, C.c_int, dptr, C.c_double, C.c_int, dptr,
                                 C.POINTER(PcgResult), C.c_char_p, C.c_size_t]
        L.oracle_residual.argtypes = [G, dptr, dptr, dptr, dptr]
        GA = C.POINTER(Grid)
        IP = C.POINTER(C.c_int)
        L.oracle_default_schedule.argtypes = [G, C.c_int, C.c_int, GA, C.c_int, IP, C.c_char_p,
                                              C.c_size_t]
        L.oracle_restrict_image.argtypes = [G, G, dptr, dptr, C.c_char_p, C.c_size_t]
        L.oracle_prolong_field.argtypes = [G, G, dptr, dptr, C.c_char_p, C.c_size_t]
        L.oracle_correct_pair.argtypes = [G, dptr, dptr, dptr, dptr, dptr, C.c_char_p, C.c_size_t]
        L.oracle_ssd.argtypes = [G, dptr, dptr, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.oracle_ncc.argtypes = [G, dptr, dptr, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
        L.oracle_simulate_pair.argtypes = [G, dptr, dptr, C.c_double, C.c_ulonglong, C.c_double,
                                           dptr, dptr, C.c_char_p, C.c_size_t]
        for nm in ("oracle_avg_x1", "oracle_diff_x1", "oracle_diff_x1_adjoint",
                   "oracle_smoother_hessian_apply"):
            getattr(L, nm).argtypes = [G, dptr, dptr]
        L.oracle_tridiag_apply.argtypes = [G, dptr, dptr, dptr, C.c_double, dptr]
        L.oracle_tridiag_solve_batched.argtypes = [G, dptr, dptr, dptr, dptr, C.c_char_p, C.c_size_t]
        L.oracle_dct_apply.argtypes = [G, dptr, C.c_double, C.c_double, dptr]
        L.oracle_distance_hessian_apply.argtypes = [G, dptr, dptr, dptr, dptr, dptr]
        L.oracle_is_strictly_feasible.argtypes = [G, dptr]
        if hasattr(L, "oracle_write_volume"):  # reference harness only
            L.oracle_write_volume.argtypes = [C.c_char_p, G, C.c_int, dptr, C.c_char_p, C.c_size_t]
            L.oracle_read_volume.argtypes = [C.c_char_p, G, IP, dptr, C.c_longlong,
                                             C.POINTER(C.c_longlong), C.c_char_p, C.c_size_t]
            L.oracle_permute_to_axis1.argtypes = [G, C.c_int, dptr, dptr, G, C.c_char_p, C.c_size_t]
            L.oracle_unpermute_field.argtypes = [G, C.c_int, dptr, dptr, G, IP, C.c_char_p,
                                                 C.c_size_t]
        L.oracle_multilevel_solve.argtypes = [G, dptr, dptr, GA, C.c_int, IP, IP, C.c_int, P, N, A,
                                              C.c_int, dptr, C.POINTER(AdmmRow), C.c_int,
                                              C.POINTER(GnRow), C.c_int,
                                              C.POINTER(abi.MultilevelStatus)]
        L.oracle_rho_schedule.argtypes = [C.c_int] + [C.c_double] * 7
        L.oracle_rho_schedule.restype = C.c_double
        L.oracle_set_threads.argtypes = [C.c_int]

    def set_threads(self, n):
        self.lib.oracle_set_threads(int(n))

    # ---- solvers -----------------------------------------------------------
    def admm_solve(self, g, ip, im, b=None, z=None, u=None, rho=0.0, params=None, cfg=None,
                   level_tag=0):
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        nf = g.faces
        bo, zo, uo = np.zeros(nf), np.zeros(nf), np.zeros(nf)
        rows = (AdmmRow * max(cfg.max_iter, 1))()
        st = SolveStatus()
        r = C.c_double(rho)
        rc = self.lib.oracle_admm_solve(C.byref(g), _p(ip), _p(im), _p(b), _p(z), _p(u), _p(bo),
                                        _p(zo), _p(uo), C.byref(r), C.byref(params), C.byref(cfg),
                                        level_tag, rows, cfg.max_iter, C.byref(st))
        return dict(rc=rc, b=bo, z=zo, u=uo, rho=r.value, stop=st.stop,
                    message=st.message.decode(), rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_iter)))

    def gn_solve(self, g, ip, im, b0=None, params=None, cfg=None, level_tag=0):
        params = params or ObjectiveParams()
        cfg = cfg or GnConfig()
        nf = g.faces
        b0 = np.zeros(nf) if b0 is None else b0
        bo = np.zeros(nf)
        rows = (GnRow * (cfg.max_outer + 1))()
        st = SolveStatus()
        rc = self.lib.oracle_gn_solve(C.byref(g), _p(ip), _p(im), _p(b0), _p(bo), C.byref(params),
                                      C.byref(cfg), level_tag, rows, cfg.max_outer + 1, C.byref(st))
        return dict(rc=rc, b=bo, stop=st.stop, message=st.message.decode(),
                    rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_outer + 1)))

    # ---- per-step ----------------------------------------------------------
    def b_update(self, g, ip, im, b, z, u, rho, params=None, cfg=None):
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        out = np.zeros(g.faces)
        st = BUpdateStats()
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_b_update(C.byref(g), _p(ip), _p(im), _p(b), _p(z), _p(u), rho,
                                      C.byref(params), C.byref(cfg), _p(out), C.byref(st), msg, 256)
        return dict(rc=rc, b=out, sqp_iters=st.sqp_iters, qp_iters=st.qp_iters,
                    kkt_violation=st.kkt_violation, max_active=st.max_active,
                    message=msg.value.decode())

    def z_update(self, g, b, u, rho, alpha):
        out = np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_z_update(C.byref(g), _p(b), _p(u), rho, alpha, _p(out), msg, 256)
        assert rc == 0, msg.value
        return out

    def dct_solve(self, g, rhs, alpha, rho):
        out = np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_dct_solve(C.byref(g), _p(rhs), alpha, rho, _p(out), msg, 256)
        return rc, out, msg.value.decode()

    def dual_update(self, g, b_new, z_new, z_old, u_old, rho, eps_abs, eps_rel):
        u = np.zeros(g.faces)
        r = DualResult()
        self.lib.oracle_dual_update(C.byref(g), _p(b_new), _p(z_new), _p(z_old), _p(u_old), rho,
                                    eps_abs, eps_rel, _p(u), C.byref(r))
        return u, dict(primal_res=r.primal_res, dual_res=r.dual_res, eps_pri=r.eps_pri,
                       eps_dual=r.eps_dual)

    def augmented_lagrangian(self, g, ip, im, b, z, u, rho, alpha):
        return self.lib.oracle_augmented_lagrangian(C.byref(g), _p(ip), _p(im), _p(b), _p(z), _p(u),
                                                    rho, alpha)

    def qp_active_set(self, n, h, gd, go, c, x0, max_iter):
        x = np.zeros(n)
        lam = np.zeros(max(n - 1, 1))
        sign = np.zeros(max(n - 1, 1), dtype=np.int32)
        it = C.c_int(0)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_qp_active_set(n, h, _p(gd), _p(go), _p(c), _p(x0), max_iter, _p(x),
                                           _p(lam), _ip(sign), C.byref(it), msg, 256)
        return dict(rc=rc, x=x, lam=lam, sign=sign, iters=it.value, message=msg.value.decode())

    def verify_qp_kkt(self, n, h, gd, go, c, x, lam, sign):
        return self.lib.oracle_verify_qp_kkt(n, h, _p(gd), _p(go), _p(c), _p(x), _p(lam), _ip(sign))

    def objective_gn(self, g, ip, im, b, params=None, need_grad=True):
        params = params or ObjectiveParams()
        grad = np.zeros(g.faces)
        res = np.zeros(g.cells)
        ev = ObjectiveEval()
        rc = self.lib.oracle_objective_gn(C.byref(g), _p(ip), _p(im), _p(b), C.byref(params),
                                          int(need_grad), C.byref(ev), _p(grad), _p(res))
        return dict(rc=rc, value=ev.value, dist=ev.dist, smooth=ev.smooth, pen=ev.pen,
                    feasible=bool(ev.feasible), grad=grad, residual=res)

    def gn_hessian_build(self, g, ip, im, b, params=None):
        params = params or ObjectiveParams()
        d, o, pd = np.zeros(g.faces), np.zeros(g.faces), np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_gn_hessian_build(C.byref(g), _p(ip), _p(im), _p(b), C.byref(params),
                                              _p(d), _p(o), _p(pd), msg, 256)
        return dict(rc=rc, diag=d, off=o, pdiag=pd, message=msg.value.decode())

    def gn_hessian_apply(self, g, ip, im, b, x, params=None):
        params = params or ObjectiveParams()
        y = np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_gn_hessian_apply(C.byref(g), _p(ip), _p(im), _p(b), C.byref(params),
                                              _p(x), _p(y), msg, 256)
        assert rc == 0, msg.value
        return y

    def precond_apply(self, g, ip, im, b, kind, r, params=None):
        params = params or ObjectiveParams()
        z = np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_precond_apply(C.byref(g), _p(ip), _p(im), _p(b), C.byref(params), kind,
                                           _p(r), _p(z), msg, 256)
        assert rc == 0, msg.value
        return z

    def pcg(self, g, ip, im, b, grad, eta, max_iters, kind=abi.PRECOND_BLOCK_JACOBI, params=None):
        params = params or ObjectiveParams()
        d = np.zeros(g.faces)
        res = PcgResult()
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_pcg(C.byref(g), _p(ip), _p(im), _p(b), C.byref(params), kind, _p(grad),
                                 eta, max_iters, _p(d), C.byref(res), msg, 256)
        return dict(rc=rc, d=d, iters=res.iters, relres=res.relres, relres_prec=res.relres_prec,
                    reached_tol=bool(res.reached_tol), message=msg.value.decode())

    # ---- image.cpp: correct_pair, ssd, ncc, simulate_pair -------------------------
    # ---- the reference's test-side helpers of the path ----
    def avg_x1(self, g, b):
        out = np.zeros(g.cells)
        assert self.lib.oracle_avg_x1(C.byref(g), _p(b), _p(out)) == 0
        return out

    def diff_x1(self, g, b):
        out = np.zeros(g.cells)
        assert self.lib.oracle_diff_x1(C.byref(g), _p(b), _p(out)) == 0
        return out

    def diff_x1_adjoint(self, g, r):
        out = np.zeros(g.faces)
        assert self.lib.oracle_diff_x1_adjoint(C.byref(g), _p(r), _p(out)) == 0
        return out

    def smoother_hessian_apply(self, g, b):
        out = np.zeros(g.faces)
        assert self.lib.oracle_smoother_hessian_apply(C.byref(g), _p(b), _p(out)) == 0
        return out

    def tridiag_apply(self, g, diag, off, x, s, y):
        y = np.array(y, dtype=np.float64)
        assert self.lib.oracle_tridiag_apply(C.byref(g), _p(diag), _p(off), _p(x), s, _p(y)) == 0
        return y

    def tridiag_solve_batched(self, g, diag, off, rhs):
        x = np.zeros(g.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_tridiag_solve_batched(C.byref(g), _p(diag), _p(off), _p(rhs), _p(x),
                                                   msg, 256)
        if rc:
            raise RuntimeError(msg.value.decode())
        return x

    def dct_apply(self, g, z, alpha, rho):
        out = np.zeros(g.faces)
        assert self.lib.oracle_dct_apply(C.byref(g), _p(z), alpha, rho, _p(out)) == 0
        return out

    def distance_hessian_apply(self, g, ip, im, b, p):
        out = np.zeros(g.faces)
        assert self.lib.oracle_distance_hessian_apply(C.byref(g), _p(ip), _p(im), _p(b), _p(p),
                                                      _p(out)) == 0
        return out

    def is_strictly_feasible(self, g, b):
        r = self.lib.oracle_is_strictly_feasible(C.byref(g), _p(b))
        assert r >= 0
        return bool(r)

    def correct_pair(self, g, ip, im, b):
        cp, cm = np.zeros(g.cells), np.zeros(g.cells)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_correct_pair(C.byref(g), _p(ip), _p(im), _p(b), _p(cp), _p(cm), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        return cp, cm

    def ssd(self, g, a, b):
        out = C.c_double()
        msg = C.create_string_buffer(256)
        if self.lib.oracle_ssd(C.byref(g), _p(a), _p(b), C.byref(out), msg, 256):
            raise ValueError(msg.value.decode())
        return out.value

    def ncc(self, g, a, b):
        out = C.c_double()
        msg = C.create_string_buffer(256)
        if self.lib.oracle_ncc(C.byref(g), _p(a), _p(b), C.byref(out), msg, 256):
            raise ValueError(msg.value.decode())
        return out.value

    def simulate_pair(self, g, truth, b_true, noise_sigma=0.0, seed=0, feas_margin=0.05):
        up, um = np.zeros(g.cells), np.zeros(g.cells)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_simulate_pair(C.byref(g), _p(truth), _p(b_true), noise_sigma, seed,
                                           feas_margin, _p(up), _p(um), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        return up, um

    # ---- volume_io (reference harness only) --------------------------------------
    def write_volume(self, path, g, kind, v):
        msg = C.create_string_buffer(256)
        if self.lib.oracle_write_volume(path.encode(), C.byref(g), kind, _p(v), msg, 256):
            raise RuntimeError(msg.value.decode())

    def read_volume(self, path):
        g, kind, n = Grid(), C.c_int(), C.c_longlong()
        msg = C.create_string_buffer(256)
        if self.lib.oracle_read_volume(path.encode(), C.byref(g), C.byref(kind), None, 0,
                                       C.byref(n), msg, 256):
            raise RuntimeError(msg.value.decode())
        v = np.zeros(n.value)
        self.lib.oracle_read_volume(path.encode(), C.byref(g), C.byref(kind), _p(v), n.value,
                                    C.byref(n), msg, 256)
        return g, kind.value, v

    def permute_to_axis1(self, g, pe_axis, img):
        out, og = np.zeros(g.cells), Grid()
        msg = C.create_string_buffer(256)
        if self.lib.oracle_permute_to_axis1(C.byref(g), pe_axis, _p(img), _p(out), C.byref(og), msg, 256):
            raise ValueError(msg.value.decode())
        return og, out

    def unpermute_field(self, g, pe_axis, b):
        out, og, kind = np.zeros(g.faces), Grid(), C.c_int()
        msg = C.create_string_buffer(256)
        if self.lib.oracle_unpermute_field(C.byref(g), pe_axis, _p(b), _p(out), C.byref(og),
                                           C.byref(kind), msg, 256):
            raise ValueError(msg.value.decode())
        return og, kind.value, out

    # ---- multilevel (multilevel.cpp) ------------------------------------------
    def default_schedule(self, fine, max_levels=4, min_cells=16):
        out = (Grid * 64)()
        n = C.c_int(0)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_default_schedule(C.byref(fine), max_levels, min_cells, out, 64,
                                              C.byref(n), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        return [out[i] for i in range(n.value)]

    def restrict_image(self, fine, coarse, img):
        out = np.zeros(coarse.cells)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_restrict_image(C.byref(fine), C.byref(coarse), _p(img), _p(out), msg,
                                            256)
        if rc:
            raise ValueError(msg.value.decode())
        return out

    def prolong_field(self, coarse, fine, b):
        out = np.zeros(fine.faces)
        msg = C.create_string_buffer(256)
        rc = self.lib.oracle_prolong_field(C.byref(coarse), C.byref(fine), _p(b), _p(out), msg, 256)
        if rc:
            raise ValueError(msg.value.decode())
        return out

    def multilevel_solve(self, fine, ip, im, levels, solver, params=None, gn_cfg=None,
                         admm_cfg=None, restart=abi.RESTART_AVERAGE, gn_max_outer=None,
                         admm_max_iter=None):
        params = params or ObjectiveParams()
        gn_cfg = gn_cfg or GnConfig()
        admm_cfg = admm_cfg or AdmmConfig()
        nlev = len(levels)
        lv = (Grid * nlev)(*levels)
        ov = lambda xs: None if xs is None else (C.c_int * nlev)(*[(-1 if x is None else x) for x in xs])  # noqa: E731
        cap_a = sum((admm_max_iter[l] if admm_max_iter and admm_max_iter[l] is not None
                     else admm_cfg.max_iter) for l in range(nlev)) + nlev
        cap_g = sum((gn_max_outer[l] if gn_max_outer and gn_max_outer[l] is not None
                     else gn_cfg.max_outer) + 1 for l in range(nlev))
        arows, grows = (AdmmRow * cap_a)(), (GnRow * cap_g)()
        b = np.zeros(fine.faces)
        st = abi.MultilevelStatus()
        rc = self.lib.oracle_multilevel_solve(C.byref(fine), _p(ip), _p(im), lv, nlev,
                                              ov(gn_max_outer), ov(admm_max_iter), solver,
                                              C.byref(params), C.byref(gn_cfg), C.byref(admm_cfg),
                                              restart, _p(b), arows, cap_a, grows, cap_g,
                                              C.byref(st))
        if rc:
            raise ValueError(st.message.decode())
        nb = levels[st.b_level].faces
        return dict(b=b[:nb], b_level=st.b_level, stop=st.stop, message=st.message.decode(),
                    admm_rows=abi.rows_to_dicts(arows, min(st.n_admm_rows, cap_a)),
                    gn_rows=abi.rows_to_dicts(grows, min(st.n_gn_rows, cap_g)))

    def residual(self, g, ip, im, b):
        r = np.zeros(g.cells)
        self.lib.oracle_residual(C.byref(g), _p(ip), _p(im), _p(b), _p(r))
        return r

    def rho_schedule(self, *args):
        return self.lib.oracle_rho_schedule(*args)


def load(kind="oracle") -> Checker:
    with _lock:
        if kind not in _libs:
            _libs[kind] = Checker(kind)
        return _libs[kind]
