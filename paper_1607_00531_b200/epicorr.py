"""Host mirror of the reference epicorr solver API over libepicorr_b200.so.

Names, argument meaning and error behaviour follow the reference's C++ entry
points (proj/include/epicorr/admm.hpp, gn_pcg.hpp, objective.hpp,
operators.hpp): `admm_solve`, `b_update`, `z_update`, `dual_update_and_
residuals`, `augmented_lagrangian`, `rho_schedule`, `qp_active_set`,
`gauss_newton_solve`, `objective_gn`, `GnHessian` parts, `pcg`. Errors the
reference throws are raised as the matching Python exception
(ValueError <- std::invalid_argument, RuntimeError <- std::runtime_error,
ArithmeticError <- std::domain_error) with the reference's message text.

Arrays: numpy float64 (host; copied through the call) or torch CUDA float64
tensors (device; used in place, EPC_MEM_DEVICE). There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from ._lib import load
from .abi import (AdmmConfig, AdmmRow, BUpdateStats, DualResult, GnConfig, GnRow, Grid,
                  ObjectiveEval, ObjectiveParams, PcgResult, SolveStatus)

_EXC = {abi.EPC_ERR_INVALID_ARGUMENT: ValueError, abi.EPC_ERR_RUNTIME: RuntimeError,
        abi.EPC_ERR_DOMAIN: ArithmeticError, abi.EPC_ERR_CUDA: OSError,
        abi.EPC_ERR_UNSUPPORTED: NotImplementedError}


class EpcError(Exception):
    pass


def _raise(code, msg):
    raise _EXC.get(code, EpcError)(msg)


def _is_dev(a):
    return a is not None and hasattr(a, "is_cuda") and a.is_cuda


class Context:
    """One device context (epc_context). `stream`: a torch.cuda.Stream, a raw
    cudaStream_t int, or None for a library-owned stream."""

    def __init__(self, device=0, stream=None):
        self.lib = load()
        h = C.c_void_p()
        raw = getattr(stream, "cuda_stream", stream)
        rc = self.lib.epc_context_create(device, C.c_void_p(raw) if raw else None, C.byref(h))
        if rc != 0:
            _raise(rc, f"epc_context_create failed (status {rc})")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.epc_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- plumbing ---------------------------------------------------------
    def _err(self):
        return self.lib.epc_last_error(self.h).decode()

    def _check(self, rc):
        if rc != 0:
            _raise(rc, self._err())

    def _mem(self, *arrays):
        dev = [_is_dev(a) for a in arrays if a is not None]
        if any(dev) and not all(dev):
            raise ValueError("mix of host and device arrays")
        if dev and dev[0]:
            # device inputs may still be in flight on torch's stream; the
            # library runs on the context's stream
            import torch
            first = next(a for a in arrays if a is not None)
            torch.cuda.current_stream(first.device).synchronize()
            return abi.EPC_MEM_DEVICE
        return abi.EPC_MEM_HOST

    @staticmethod
    def _ptr(a):
        if a is None:
            return None
        if _is_dev(a):
            assert a.dtype.__str__() == "torch.float64" and a.is_contiguous()
            return C.c_void_p(a.data_ptr())
        assert isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data)

    def _like(self, ref, n):
        if _is_dev(ref):
            import torch
            return torch.empty(n, dtype=torch.float64, device=ref.device)
        return np.zeros(n)

    def set_stream(self, stream):
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self.lib.epc_set_stream(self.h, C.c_void_p(raw) if raw else None))

    def launch_count(self):
        return self.lib.epc_launch_count(self.h)

    def reset_launch_count(self):
        self.lib.epc_reset_launch_count(self.h)

    def profile(self, on=True):
        self.lib.epc_profile_enable(self.h, int(on))

    def profile_reset(self):
        self.lib.epc_profile_reset(self.h)

    def set_mode(self, bits):
        self._check(self.lib.epc_set_mode(self.h, int(bits)))

    BSTEP_PHASES = ["model", "fval_sums", "factor", "solves", "qp_rest", "kkt", "step_sums",
                    "line_search", "clamp_store", "fetch"]

    def bstep_timing(self):
        out = (C.c_longlong * 10)()
        self._check(self.lib.epc_bstep_timing(self.h, out))
        return dict(zip(self.BSTEP_PHASES, list(out)))

    BSTEP_COUNTERS = ["ls_trials", "ls_undecided", "stop_undecided", "ls_failed", "ls_searches",
                      "fval_exact", "acc0", "acc1", "acc2_3", "acc4_7", "acc8_15", "acc16_31",
                      "acc32_39", "fail", "schur_n", "schur_na", "schur_na2", "schur_na3"]
    MODE_BSTEP_TIMING = 1
    MODE_BSTEP_CHAINED = 1 << 13
    MODE_EXACT_SUMS = 1 << 14
    MODE_DEVICE_LOOP = 1 << 15

    def guard_check(self):
        """First scratch slot whose guard zones were overwritten, or -1
        (contexts created with EPC_GUARD=1)."""
        b = C.c_int(-1)
        self._check(self.lib.epc_guard_check(self.h, C.byref(b)))
        return b.value

    def admm_counters(self):
        """Cumulative (decisions certified from the tree sums, decisions taken
        on the reference's exact sequential sums, SQP iterations, QP iterations)."""
        out = (C.c_longlong * 4)()
        self._check(self.lib.epc_admm_counters(self.h, out))
        return tuple(int(x) for x in out)

    def bstep_counters(self):
        out = (C.c_longlong * 18)()
        self._check(self.lib.epc_bstep_counters(self.h, out))
        return dict(zip(self.BSTEP_COUNTERS, list(out)))

    def profile_read(self):
        cap = 64
        names = (C.c_char_p * cap)()
        ms = (C.c_double * cap)()
        n = (C.c_long * cap)()
        cnt = C.c_int(0)
        self.lib.epc_profile_read(self.h, names, ms, n, cap, C.byref(cnt))
        return {names[i].decode(): (ms[i], n[i]) for i in range(min(cnt.value, cap))}

    # ---- ADMM -------------------------------------------------------------
    def admm_solve(self, g: Grid, ip, im, b=None, z=None, u=None, rho=0.0, params=None, cfg=None,
                   level_tag=0):
        """admm_solve (admm.hpp:127-129). Returns dict(b, z, u, rho, stop, message, rows)."""
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        mem = self._mem(ip, im, b, z, u)
        nf = g.faces
        bo, zo, uo = self._like(ip, nf), self._like(ip, nf), self._like(ip, nf)
        rows = (AdmmRow * max(cfg.max_iter, 1))()
        st = SolveStatus()
        r = C.c_double(rho)
        rc = self.lib.epc_admm_solve(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                     self._ptr(b), self._ptr(z), self._ptr(u), self._ptr(bo),
                                     self._ptr(zo), self._ptr(uo), C.byref(r), C.byref(params),
                                     C.byref(cfg), level_tag, rows, cfg.max_iter, C.byref(st))
        if rc != 0:
            _raise(rc, self._err() or st.message.decode())
        return dict(b=bo, z=zo, u=uo, rho=r.value, stop=st.stop, message=st.message.decode(),
                    rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_iter)))

    @staticmethod
    def _ptr32(a):
        if a is None:
            return None
        if _is_dev(a):
            assert str(a.dtype) == "torch.float32" and a.is_contiguous()
            return C.c_void_p(a.data_ptr())
        assert isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data)

    def admm_solve_f32(self, g: Grid, ip, im, b=None, z=None, u=None, rho=0.0, params=None,
                       cfg=None, level_tag=0):
        """fp32 variant of admm_solve (epc_admm_solve_f32; not bitwise).
        ip/im/b/z/u: float32 numpy arrays or CUDA tensors. Returns the admm_solve dict."""
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        mem = self._mem(ip, im, b, z, u)
        nf = g.faces
        if _is_dev(ip):
            import torch
            bo, zo, uo = (torch.empty(nf, dtype=torch.float32, device=ip.device) for _ in range(3))
        else:
            bo, zo, uo = (np.zeros(nf, dtype=np.float32) for _ in range(3))
        rows = (AdmmRow * max(cfg.max_iter, 1))()
        st = SolveStatus()
        r = C.c_double(rho)
        P32 = self._ptr32
        rc = self.lib.epc_admm_solve_f32(self.h, C.byref(g), mem, P32(ip), P32(im), P32(b), P32(z),
                                         P32(u), P32(bo), P32(zo), P32(uo), C.byref(r),
                                         C.byref(params), C.byref(cfg), level_tag, rows,
                                         cfg.max_iter, C.byref(st))
        if rc != 0:
            _raise(rc, st.message.decode() or self._err())
        return dict(b=bo, z=zo, u=uo, rho=r.value, stop=st.stop, message=st.message.decode(),
                    rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_iter)))

    def slab_admm_solve(self, comm, rank, world, g: Grid, ip, im, b=None, z=None, u=None, rho=0.0,
                        params=None, cfg=None, level_tag=0):
        """epc_slab_admm_solve: this rank's k-slab of one volume, NCCL between
        the steps (comm: NcclComm or None at world 1). ip/im/b/z/u: this
        rank's slabs as CUDA tensors. Returns the admm_solve dict (slabs)."""
        import torch
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        m1, m2, m3 = g.m
        base, extra = divmod(m3, world)
        mk = base + (1 if rank < extra else 0)
        nf = (m1 + 1) * m2 * mk
        bo, zo, uo = (torch.empty(nf, dtype=torch.float64, device=ip.device) for _ in range(3))
        rows = (AdmmRow * max(cfg.max_iter, 1))()
        st = SolveStatus()
        r = C.c_double(rho)
        torch.cuda.synchronize(ip.device)
        P = self._ptr
        rc = self.lib.epc_slab_admm_solve(self.h, comm.h if comm is not None else None, rank, world,
                                          C.byref(g), P(ip), P(im), P(b), P(z), P(u), P(bo), P(zo),
                                          P(uo), C.byref(r), C.byref(params), C.byref(cfg), level_tag,
                                          rows, cfg.max_iter, C.byref(st))
        if rc != 0:
            _raise(rc, st.message.decode() or self._err())
        return dict(b=bo, z=zo, u=uo, rho=r.value, stop=st.stop, message=st.message.decode(),
                    rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_iter)))

    def admm_solve_batch(self, g: Grid, npairs, ip, im, rho=None, params=None, cfg=None,
                         level_tag=0, b=None, z=None, u=None):
        """npairs independent admm_solve calls on one grid in the same kernels
        (pair-major arrays; b/z/u: optional warm starts for every pair, rho:
        per-pair start values, <= 0 selects rho0). Returns dict(b, z, u, pairs)."""
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        mem = self._mem(ip, im, b, z, u)
        nf = g.faces * npairs
        bo, zo, uo = self._like(ip, nf), self._like(ip, nf), self._like(ip, nf)
        rows = (AdmmRow * (max(cfg.max_iter, 1) * npairs))()
        st = (SolveStatus * npairs)()
        rh = (C.c_double * npairs)(*([0.0] * npairs if rho is None else rho))
        rc = self.lib.epc_admm_solve_batch(self.h, C.byref(g), npairs, mem, self._ptr(ip),
                                           self._ptr(im), self._ptr(b), self._ptr(z), self._ptr(u),
                                           self._ptr(bo),
                                           self._ptr(zo), self._ptr(uo), rh, C.byref(params),
                                           C.byref(cfg), level_tag, rows, cfg.max_iter, st)
        if rc != 0:
            _raise(rc, self._err())
        out = []
        for q in range(npairs):
            rr = [rows[q * cfg.max_iter + i] for i in range(min(st[q].nrows, cfg.max_iter))]
            out.append(dict(stop=st[q].stop, message=st[q].message.decode(), rho=rh[q],
                            rows=[{k: getattr(x, k) for k, _ in x._fields_} for x in rr]))
        return dict(b=bo, z=zo, u=uo, pairs=out)

    def b_update(self, g, ip, im, b, z, u, rho, params=None, cfg=None):
        params = params or ObjectiveParams()
        cfg = cfg or AdmmConfig()
        mem = self._mem(ip, im, b, z, u)
        out = self._like(b, g.faces)
        st = BUpdateStats()
        self._check(self.lib.epc_b_update(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                          self._ptr(b), self._ptr(z), self._ptr(u), rho,
                                          C.byref(params), C.byref(cfg), self._ptr(out),
                                          C.byref(st)))
        return dict(b=out, sqp_iters=st.sqp_iters, qp_iters=st.qp_iters,
                    kkt_violation=st.kkt_violation, max_active=st.max_active)

    def z_update(self, g, b, u, rho, alpha):
        mem = self._mem(b, u)
        out = self._like(b, g.faces)
        self._check(self.lib.epc_z_update(self.h, C.byref(g), mem, self._ptr(b), self._ptr(u), rho,
                                          alpha, self._ptr(out)))
        return out

    def dct_solve(self, g, rhs, alpha, rho):
        mem = self._mem(rhs)
        out = self._like(rhs, g.faces)
        self._check(self.lib.epc_dct_solve(self.h, C.byref(g), mem, self._ptr(rhs), alpha, rho,
                                           self._ptr(out)))
        return out

    def dual_update(self, g, b_new, z_new, z_old, u_old, rho, eps_abs, eps_rel):
        mem = self._mem(b_new, z_new, z_old, u_old)
        u = self._like(b_new, g.faces)
        r = DualResult()
        self._check(self.lib.epc_dual_update(self.h, C.byref(g), mem, self._ptr(b_new),
                                             self._ptr(z_new), self._ptr(z_old), self._ptr(u_old),
                                             rho, eps_abs, eps_rel, self._ptr(u), C.byref(r)))
        return u, dict(primal_res=r.primal_res, dual_res=r.dual_res, eps_pri=r.eps_pri,
                       eps_dual=r.eps_dual)

    def augmented_lagrangian(self, g, ip, im, b, z, u, rho, alpha):
        mem = self._mem(ip, im, b, z, u)
        out = C.c_double()
        self._check(self.lib.epc_augmented_lagrangian(self.h, C.byref(g), mem, self._ptr(ip),
                                                      self._ptr(im), self._ptr(b), self._ptr(z),
                                                      self._ptr(u), rho, alpha, C.byref(out)))
        return out.value

    def rho_schedule(self, *args):
        return self.lib.epc_rho_schedule(*args)

    def qp_active_set_batch(self, n, h, gd, go, c, x0, max_iter):
        """Many independent column QPs (qp_active_set + verify_qp_kkt)."""
        gd, go, c, x0 = (np.ascontiguousarray(a, dtype=np.float64) for a in (gd, go, c, x0))
        nqp = gd.size // n
        x = np.zeros(nqp * n)
        lam = np.zeros(nqp * (n - 1))
        sign = np.zeros(nqp * (n - 1), dtype=np.int32)
        iters = np.zeros(nqp, dtype=np.int32)
        kkt = np.zeros(nqp)
        status = np.zeros(nqp, dtype=np.int32)
        P = lambda a: C.c_void_p(a.ctypes.data)
        self._check(self.lib.epc_qp_active_set_batch(self.h, nqp, n, h, P(gd), P(go), P(c), P(x0),
                                                     max_iter, P(x), P(lam), P(sign), P(iters),
                                                     P(kkt), P(status)))
        return dict(x=x.reshape(nqp, n), lam=lam.reshape(nqp, n - 1),
                    sign=sign.reshape(nqp, n - 1), iters=iters, kkt=kkt, status=status,
                    message=self._err())

    def residual(self, g, ip, im, b):
        mem = self._mem(ip, im, b)
        r = self._like(ip, g.cells)
        self._check(self.lib.epc_residual(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                          self._ptr(b), self._ptr(r)))
        return r

    # ---- GN-PCG -----------------------------------------------------------
    def gn_solve(self, g, ip, im, b0=None, params=None, cfg=None, level_tag=0):
        """gauss_newton_solve (gn_pcg.hpp:81-83)."""
        params = params or ObjectiveParams()
        cfg = cfg or GnConfig()
        mem = self._mem(ip, im, b0)
        if b0 is None:
            b0 = self._like(ip, g.faces)
            if not _is_dev(b0):
                b0[:] = 0.0
            else:
                b0.zero_()
        bo = self._like(ip, g.faces)
        rows = (GnRow * (cfg.max_outer + 1))()
        st = SolveStatus()
        rc = self.lib.epc_gn_solve(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                   self._ptr(b0), self._ptr(bo), C.byref(params), C.byref(cfg),
                                   level_tag, rows, cfg.max_outer + 1, C.byref(st))
        if rc != 0:
            _raise(rc, self._err())
        return dict(b=bo, stop=st.stop, message=st.message.decode(),
                    rows=abi.rows_to_dicts(rows, min(st.nrows, cfg.max_outer + 1)))

    # ---- the reference's test-side helpers of the path ---------
    def _unary(self, fn, g, a, n_out):
        mem = self._mem(a)
        out = self._like(a, n_out)
        self._check(getattr(self.lib, fn)(self.h, C.byref(g), mem, self._ptr(a), self._ptr(out)))
        return out

    def avg_x1(self, g, b):
        """avg_x1 (operators.cpp:27-37): faces -> cells."""
        return self._unary("epc_avg_x1", g, b, g.cells)

    def diff_x1(self, g, b):
        """diff_x1 (operators.cpp:40-52): faces -> cells."""
        return self._unary("epc_diff_x1", g, b, g.cells)

    def diff_x1_adjoint(self, g, r):
        """diff_x1_adjoint (operators.cpp:54-68): cells -> faces."""
        return self._unary("epc_diff_x1_adjoint", g, r, g.faces)

    def smoother_hessian_apply(self, g, b):
        """smoother_hessian_apply (operators.cpp:141-183)."""
        return self._unary("epc_smoother_hessian_apply", g, b, g.faces)

    def tridiag_apply(self, g, diag, off, x, s, y):
        """TridiagBlocks::apply (operators.cpp:202-216): returns y + s T x."""
        mem = self._mem(diag, off, x, y)
        yo = y.clone() if _is_dev(y) else np.array(y, dtype=np.float64)
        self._check(self.lib.epc_tridiag_apply(self.h, C.byref(g), mem, self._ptr(diag),
                                               self._ptr(off), self._ptr(x), s, self._ptr(yo)))
        return yo

    def tridiag_solve_batched(self, g, diag, off, rhs):
        """tridiag_solve_batched (operators.cpp:264-273)."""
        mem = self._mem(diag, off, rhs)
        x = self._like(rhs, g.faces)
        self._check(self.lib.epc_tridiag_solve_batched(self.h, C.byref(g), mem, self._ptr(diag),
                                                       self._ptr(off), self._ptr(rhs), self._ptr(x)))
        return x

    def gn_stencil_apply(self, g, diag, off, w2, w3, x):
        """GnHessian::apply (objective.cpp:302-331) from the column part."""
        mem = self._mem(diag, off, x)
        y = self._like(x, g.faces)
        self._check(self.lib.epc_gn_stencil_apply(self.h, C.byref(g), mem, self._ptr(diag),
                                                  self._ptr(off), w2, w3, self._ptr(x), self._ptr(y)))
        return y

    def gn_cross_diag_add(self, g, diag, w2, w3):
        """GnHessian::preconditioner_blocks().diag / full_diagonal() (objective.cpp:333-348)."""
        mem = self._mem(diag)
        out = self._like(diag, g.faces)
        self._check(self.lib.epc_gn_cross_diag_add(self.h, C.byref(g), mem, self._ptr(diag), w2, w3,
                                                   self._ptr(out)))
        return out

    def jacobi_apply(self, diag, r):
        """The Jacobi preconditioner's apply, z = r / diag (gn_pcg.cpp:41-47)."""
        mem = self._mem(diag, r)
        n = len(r)
        z = self._like(r, n)
        self._check(self.lib.epc_jacobi_apply(self.h, n, mem, self._ptr(diag), self._ptr(r),
                                              self._ptr(z)))
        return z

    def dct_apply(self, g, z, alpha, rho):
        """DctCoupledSolver::apply (operators.cpp:420-446): Gt z."""
        mem = self._mem(z)
        out = self._like(z, g.faces)
        self._check(self.lib.epc_dct_apply(self.h, C.byref(g), mem, self._ptr(z), alpha, rho,
                                           self._ptr(out)))
        return out

    def distance_hessian_apply(self, g, ip, im, b, p):
        """DistanceEval::hessian_apply (objective.cpp:128-147) at b."""
        mem = self._mem(ip, im, b, p)
        out = self._like(p, g.faces)
        self._check(self.lib.epc_distance_hessian_apply(self.h, C.byref(g), mem, self._ptr(ip),
                                                        self._ptr(im), self._ptr(b), self._ptr(p),
                                                        self._ptr(out)))
        return out

    def is_strictly_feasible(self, g, b):
        """is_strictly_feasible (objective.cpp:35-37)."""
        f = C.c_int(0)
        self._check(self.lib.epc_is_strictly_feasible(self.h, C.byref(g), self._mem(b),
                                                      self._ptr(b), C.byref(f)))
        return bool(f.value)

    # ---- either side of the solve (image.hpp:62-86) ------------------------------
    def correct_pair(self, g, ip, im, b):
        """correct_pair (image.cpp:226-253) -> (corrected plus, corrected minus)."""
        mem = self._mem(ip, im, b)
        cp, cm = self._like(ip, g.cells), self._like(ip, g.cells)
        self._check(self.lib.epc_correct_pair(self.h, C.byref(g), mem, self._ptr(ip),
                                              self._ptr(im), self._ptr(b), self._ptr(cp),
                                              self._ptr(cm)))
        return cp, cm

    def ssd(self, g, a, b):
        """ssd (image.cpp:255-263)."""
        out = C.c_double()
        self._check(self.lib.epc_ssd(self.h, C.byref(g), self._mem(a, b), self._ptr(a),
                                     self._ptr(b), C.byref(out)))
        return out.value

    def ncc(self, g, a, b):
        """ncc (image.cpp:265-283)."""
        out = C.c_double()
        self._check(self.lib.epc_ncc(self.h, C.byref(g), self._mem(a, b), self._ptr(a),
                                     self._ptr(b), C.byref(out)))
        return out.value

    def simulate_pair(self, g, truth, b_true, noise_sigma=0.0, seed=0, feas_margin=0.05):
        """simulate_pair (image.cpp:187-224) -> (I+, I-)."""
        mem = self._mem(truth, b_true)
        up, um = self._like(truth, g.cells), self._like(truth, g.cells)
        self._check(self.lib.epc_simulate_pair(self.h, C.byref(g), mem, self._ptr(truth),
                                               self._ptr(b_true), noise_sigma, seed, feas_margin,
                                               self._ptr(up), self._ptr(um)))
        return up, um

    # ---- phase-encoding permutation (volume_io.hpp:45-53) -----------------------
    def permute_to_axis1(self, g, pe_axis, img):
        """permute_to_axis1 (volume_io.cpp:203-209) -> (grid, cells)."""
        out, og = self._like(img, g.cells), Grid()
        self._check(self.lib.epc_permute_to_axis1(self.h, C.byref(g), pe_axis, self._mem(img),
                                                  self._ptr(img), self._ptr(out), C.byref(og)))
        return og, out

    def unpermute_field(self, g, pe_axis, b):
        """unpermute_field (volume_io.cpp:211-223) -> (grid, kind, faces)."""
        out, og, kind = self._like(b, g.faces), Grid(), C.c_int()
        self._check(self.lib.epc_unpermute_field(self.h, C.byref(g), pe_axis, self._mem(b),
                                                 self._ptr(b), self._ptr(out), C.byref(og),
                                                 C.byref(kind)))
        return og, kind.value, out

    # ---- multilevel (multilevel.hpp:13-63) -------------------------------------
    def restrict_image(self, fine, coarse, img):
        """restrict_image (multilevel.cpp:98-131)."""
        mem = self._mem(img)
        out = self._like(img, coarse.cells)
        self._check(self.lib.epc_restrict_image(self.h, C.byref(fine), C.byref(coarse), mem,
                                                self._ptr(img), self._ptr(out)))
        return out

    def prolong_field(self, coarse, fine, b):
        """prolong_field (multilevel.cpp:157-203)."""
        mem = self._mem(b)
        out = self._like(b, fine.faces)
        self._check(self.lib.epc_prolong_field(self.h, C.byref(coarse), C.byref(fine), mem,
                                               self._ptr(b), self._ptr(out)))
        return out

    def multilevel_solve(self, fine, ip, im, levels, solver, params=None, gn_cfg=None,
                         admm_cfg=None, restart=abi.RESTART_AVERAGE, gn_max_outer=None,
                         admm_max_iter=None):
        """multilevel_solve (multilevel.hpp:57-63). levels: coarse -> fine Grid
        list (e.g. default_schedule(fine)); solver abi.SOLVER_GN / SOLVER_ADMM;
        per-level overrides as lists (None entries: no override). Returns
        dict(b, b_level, stop, message, admm_rows, gn_rows)."""
        params = params or ObjectiveParams()
        gn_cfg = gn_cfg or GnConfig()
        admm_cfg = admm_cfg or AdmmConfig()
        nlev = len(levels)
        mem = self._mem(ip, im)
        lv = (Grid * nlev)(*levels)
        ov = lambda xs: None if xs is None else (C.c_int * nlev)(*[(-1 if x is None else x) for x in xs])  # noqa: E731
        cap_a = sum((admm_max_iter[l] if admm_max_iter and admm_max_iter[l] is not None
                     else admm_cfg.max_iter) for l in range(nlev)) + nlev
        cap_g = sum((gn_max_outer[l] if gn_max_outer and gn_max_outer[l] is not None
                     else gn_cfg.max_outer) + 1 for l in range(nlev))
        arows, grows = (AdmmRow * cap_a)(), (GnRow * cap_g)()
        b = self._like(ip, fine.faces)
        st = abi.MultilevelStatus()
        rc = self.lib.epc_multilevel_solve(self.h, C.byref(fine), mem, self._ptr(ip),
                                           self._ptr(im), lv, nlev, ov(gn_max_outer),
                                           ov(admm_max_iter), solver, C.byref(params),
                                           C.byref(gn_cfg), C.byref(admm_cfg), restart,
                                           self._ptr(b), arows, cap_a, grows, cap_g, C.byref(st))
        if rc != 0:
            _raise(rc, st.message.decode() or self._err())
        nb = levels[st.b_level].faces
        return dict(b=b[:nb], b_level=st.b_level, stop=st.stop, message=st.message.decode(),
                    admm_rows=abi.rows_to_dicts(arows, min(st.n_admm_rows, cap_a)),
                    gn_rows=abi.rows_to_dicts(grows, min(st.n_gn_rows, cap_g)))

    def objective_gn(self, g, ip, im, b, params=None, need_grad=True):
        params = params or ObjectiveParams()
        mem = self._mem(ip, im, b)
        grad = self._like(b, g.faces)
        res = self._like(b, g.cells)
        ev = ObjectiveEval()
        self._check(self.lib.epc_objective_gn(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                              self._ptr(b), C.byref(params), int(need_grad),
                                              C.byref(ev), self._ptr(grad), self._ptr(res)))
        return dict(value=ev.value, dist=ev.dist, smooth=ev.smooth, pen=ev.pen,
                    feasible=bool(ev.feasible), grad=grad, residual=res)

    def gn_hessian_build(self, g, ip, im, b, params=None):
        params = params or ObjectiveParams()
        mem = self._mem(ip, im, b)
        d, o, pd = (self._like(b, g.faces) for _ in range(3))
        self._check(self.lib.epc_gn_hessian_build(self.h, C.byref(g), mem, self._ptr(ip),
                                                  self._ptr(im), self._ptr(b), C.byref(params),
                                                  self._ptr(d), self._ptr(o), self._ptr(pd)))
        return dict(diag=d, off=o, pdiag=pd)

    def gn_hessian_apply(self, g, ip, im, b, x, params=None):
        params = params or ObjectiveParams()
        mem = self._mem(ip, im, b, x)
        y = self._like(b, g.faces)
        self._check(self.lib.epc_gn_hessian_apply(self.h, C.byref(g), mem, self._ptr(ip),
                                                  self._ptr(im), self._ptr(b), C.byref(params),
                                                  self._ptr(x), self._ptr(y)))
        return y

    def precond_apply(self, g, ip, im, b, kind, r, params=None):
        params = params or ObjectiveParams()
        mem = self._mem(ip, im, b, r)
        z = self._like(b, g.faces)
        self._check(self.lib.epc_precond_apply(self.h, C.byref(g), mem, self._ptr(ip),
                                               self._ptr(im), self._ptr(b), C.byref(params), kind,
                                               self._ptr(r), self._ptr(z)))
        return z

    def pcg(self, g, ip, im, b, grad, eta, max_iters, kind=abi.PRECOND_BLOCK_JACOBI, params=None):
        params = params or ObjectiveParams()
        mem = self._mem(ip, im, b, grad)
        d = self._like(b, g.faces)
        res = PcgResult()
        self._check(self.lib.epc_pcg(self.h, C.byref(g), mem, self._ptr(ip), self._ptr(im),
                                     self._ptr(b), C.byref(params), kind, self._ptr(grad), eta,
                                     max_iters, self._ptr(d), C.byref(res)))
        return dict(d=d, iters=res.iters, relres=res.relres, relres_prec=res.relres_prec,
                    reached_tol=bool(res.reached_tol))


_default = None


def admm_solve_batch_devices(contexts, g: Grid, npairs, ip, im, cfg=None, params=None, rho=None,
                             b=None, z=None, u=None, level_tag=0):
    """epc_admm_solve_batch_devices: npairs pairs (pair-major host arrays)
    split over the contexts' devices, solved concurrently (no collective).
    Returns dict(b, z, u, pairs) like Context.admm_solve_batch."""
    lib = load()
    params = params or ObjectiveParams()
    cfg = cfg or AdmmConfig()
    nf = g.faces * npairs
    bo, zo, uo = np.zeros(nf), np.zeros(nf), np.zeros(nf)
    rows = (AdmmRow * (max(cfg.max_iter, 1) * npairs))()
    st = (SolveStatus * npairs)()
    rh = (C.c_double * npairs)(*([0.0] * npairs if rho is None else rho))
    hs = (C.c_void_p * len(contexts))(*[c.h.value for c in contexts])
    P = lambda a: None if a is None else C.c_void_p(np.ascontiguousarray(a, np.float64).ctypes.data)
    keep = [np.ascontiguousarray(a, np.float64) for a in (ip, im, b, z, u) if a is not None]
    rc = lib.epc_admm_solve_batch_devices(hs, len(contexts), C.byref(g), npairs, P(ip), P(im), P(b),
                                          P(z), P(u), C.c_void_p(bo.ctypes.data),
                                          C.c_void_p(zo.ctypes.data), C.c_void_p(uo.ctypes.data), rh,
                                          C.byref(params), C.byref(cfg), level_tag, rows,
                                          cfg.max_iter, st)
    del keep
    if rc != 0:
        _raise(rc, contexts[0]._err())
    out = []
    for q in range(npairs):
        rr = [rows[q * cfg.max_iter + i] for i in range(min(st[q].nrows, cfg.max_iter))]
        out.append(dict(stop=st[q].stop, message=st[q].message.decode(), rho=rh[q],
                        rows=[{k: getattr(x, k) for k, _ in x._fields_} for x in rr]))
    return dict(b=bo, z=zo, u=uo, pairs=out)


def nccl_unique_id() -> bytes:
    """epc_nccl_unique_id: 128 bytes to broadcast from rank 0."""
    buf = C.create_string_buffer(128)
    rc = load().epc_nccl_unique_id(buf)
    if rc != 0:
        _raise(rc, "epc_nccl_unique_id failed (NCCL unavailable?)")
    return buf.raw


class NcclComm:
    """An NCCL communicator made by the library (epc_nccl_comm_create)."""

    def __init__(self, device, world, rank, uid: bytes):
        self.lib = load()
        self.h = C.c_void_p()
        rc = self.lib.epc_nccl_comm_create(device, world, rank, uid, C.byref(self.h))
        if rc != 0:
            _raise(rc, "epc_nccl_comm_create failed")
        self.world, self.rank = world, rank

    def close(self):
        if self.h:
            self.lib.epc_nccl_comm_destroy(self.h)
            self.h = C.c_void_p()


def context(device=0):
    global _default
    if _default is None:
        _default = Context(device)
    return _default


def default_schedule(fine, max_levels=4, min_cells=16):
    """default_schedule (multilevel.cpp:22-41): coarse -> fine Grid list."""
    L = load()
    out = (Grid * 64)()
    n = C.c_int(0)
    rc = L.epc_default_schedule(C.byref(fine), max_levels, min_cells, out, 64, C.byref(n))
    if rc != 0:
        _raise(rc, "default_schedule: invalid grid")
    return [out[i] for i in range(n.value)]


def write_volume(path, g, kind, v):
    """write_volume (volume_io.cpp:68-100): EPIVOL 1, float32 payload."""
    rc = load().epc_write_volume(str(path).encode(), C.byref(g), kind,
                                 C.c_void_p(np.ascontiguousarray(v, dtype=np.float64).ctypes.data))
    if rc != 0:
        _raise(rc, f"write_volume: cannot write {path}")


def read_volume(path):
    """read_volume (volume_io.cpp:102-171) -> (grid, kind, values)."""
    L = load()
    g, kind, n = Grid(), C.c_int(), C.c_longlong()
    rc = L.epc_read_volume(str(path).encode(), C.byref(g), C.byref(kind), None, 0, C.byref(n))
    if rc != 0:
        _raise(rc, f"read_volume: cannot read {path}")
    v = np.zeros(n.value)
    rc = L.epc_read_volume(str(path).encode(), C.byref(g), C.byref(kind),
                           C.c_void_p(v.ctypes.data), n.value, C.byref(n))
    if rc != 0:
        _raise(rc, f"read_volume: cannot read {path}")
    return g, kind.value, v
