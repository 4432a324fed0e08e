"""Gauss-Newton-PCG in k-slabs over several GPUs (GN row).

Same decomposition as dist_admm: rank r owns face layers [k0, k0 + mk). GN
couples k only through the stencils (objective_gn's D3 terms and
GnHessian::apply's w3 coupling, objective.cpp:231-331), so every vector is
held *extended* with one halo layer to each neighbour and the ranks exchange
  * one layer of p each way per PCG iteration (the 7-point stencil),
  * one layer of the search direction per GN iteration (trial points b + t d
    are then formed locally, halos included),
and all-gather the partial sums (pq; rr and rz; the objective's sums and
maxima; the dots of the stopping tests). The block-Jacobi preconditioner is
per column, hence local. The host logic restates gauss_newton_solve
(gn_pcg.cpp:197-292), pcg (:92-131) and wolfe_linesearch (:141-195) exactly
as api.cu's epc_gn_solve does; the device arithmetic is the single-GPU
path's, only the order of the cross-rank sums differs (rank order on every
rank, so the replicated decisions are identical).
"""
from __future__ import annotations

import ctypes as C
import math
import time

from . import abi
from .dist_admm import Slabs  # noqa: F401  (same slab bookkeeping)

STOP_CONVERGED, STOP_MAX_ITER, STOP_LS_FAILURE, STOP_ERROR = 0, 1, 2, 3


class Obj:
    __slots__ = ("value", "dphi", "d1max", "feasible")


def _ext_layout(grid, slabs, rank):
    k0, mk = slabs.k_range(rank)
    lo = 1 if k0 > 0 else 0
    hi = 1 if k0 + mk < slabs.m3 else 0
    return k0, mk, lo, hi


def gn_rank(backend, grid, slabs, rank, ip_ext, im_ext, b0_ext=None, cfg=None, params=None,
            level_tag=0):
    """One rank of the distributed gauss_newton_solve (a generator yielding
    collective requests; run it with dist_admm.run_torch / run_lockstep).
    ip_ext / im_ext: the rank's cells for layers k0-lo .. k0+mk+hi-1;
    b0_ext: optional start (extended faces). Returns dict(b (owned faces),
    rows, stop, message)."""
    cfg = cfg or abi.GnConfig()
    P = params or abi.ObjectiveParams()
    k0, mk, lo, hi = _ext_layout(grid, slabs, rank)
    layer = slabs.n1 * slabs.m2
    ne = (lo + mk + hi) * layer
    o0, o1 = lo * layer, (lo + mk) * layer
    V = grid.h[0] * grid.h[1] * grid.h[2]
    ext = (grid, k0, mk, lo, hi)
    vec = backend.zeros
    b, bnew, trial, zero = vec(ne), vec(ne), vec(ne), vec(ne)
    grad, tgrad, dirv = vec(ne), vec(ne), vec(ne)
    r, z, p, q = vec(ne), vec(ne), vec(ne), vec(ne)
    if b0_ext is not None:
        backend.copy(b, b0_ext)
    own = lambda x: backend.view(x, o0, o1 - o0)  # noqa: E731

    def gsum(vals):
        allv = yield ("gather", list(vals))
        return allv

    def objective(x, need_grad, g_out, d_ext, keep_jac=False):
        o8 = backend.gn_objective(ext, P, ip_ext, im_ext, x, need_grad, g_out, d_ext, keep_jac)
        allv = yield from gsum(o8)
        sr = sd = sp = s2 = s3 = sgd = 0.0
        d1 = am = 0.0
        for v in allv:
            sr += v[0]
            sd += v[1]
            sp += v[2]
            d1 = v[3] if d1 < v[3] else d1
            s2 += v[4]
            s3 += v[5]
            sgd += v[6]
            am = v[7] if am < v[7] else am
        o = Obj()
        o.d1max = d1
        o.feasible = P.beta == 0.0 or d1 <= 1.0 - 1e-10   # objective.cpp:237-240
        if P.enforce_linf_box:  # within_linf_box (objective.cpp:39-44)
            ext_len = (grid.m[0] * grid.h[0], grid.m[1] * grid.h[1], grid.m[2] * grid.h[2])
            diam2 = 0.0
            for a in range(grid.dim):
                diam2 += ext_len[a] * ext_len[a]
            if not (am <= 2.0 * math.sqrt(diam2)):
                o.feasible = False
        if not o.feasible:
            o.value, o.dphi = math.inf, 0.0
            return o
        dist = 0.5 * V * sr
        s = sd
        s += s2
        if grid.dim == 3:
            s += s3
        smooth = 0.5 * V * s
        pen = P.beta * V * sp if P.beta > 0.0 else 0.0
        o.value = dist + P.alpha * smooth + pen
        o.dphi = sgd
        return o

    def dot(a, bvec):
        ab_bb = backend.dot(own(a), own(bvec))
        allv = yield from gsum(ab_bb)
        s0 = s1 = 0.0
        for v in allv:
            s0 += v[0]
            s1 += v[1]
        return s0, s1

    def pcg(eta, max_iters):
        """gn_pcg.cpp:92-131 with H = GnHessian(b), M = cfg.precond; the
        solution goes to dirv (extended; owned part valid)."""
        backend.fill0(dirv)
        gg = backend.negate(own(grad), own(r))
        allv = yield from gsum([gg])
        gnorm = math.sqrt(sum(v[0] for v in allv))
        if gnorm == 0.0:
            return 0, 0.0, 0.0, True
        rr_rz = backend.gn_update(ext, P, cfg.precond, 0.0, False, dirv, r, z, None, None)
        allv = yield from gsum(rr_rz)
        rz = 0.0
        for v in allv:
            rz += v[1]
        prec0 = math.sqrt(rz if rz > 0.0 else 0.0)
        beta, iters, relres, relres_prec, reached = 0.0, 0, 0.0, 0.0, False
        for it in range(max_iters):
            if it == 0:
                backend.copy(own(p), own(z))
            else:
                backend.axpy(own(z), beta, own(p), own(p))   # p = z + beta p
            yield ("halo2", p, o0, o1, layer, lo, hi)
            pq = backend.gn_hv(ext, P, p, q)
            allv = yield from gsum([pq])
            pqs = sum(v[0] for v in allv)
            if not (pqs > 0.0):
                raise RuntimeError("pcg: nonpositive curvature encountered")
            alpha = rz / pqs
            rr_rz = backend.gn_update(ext, P, cfg.precond, alpha, True, dirv, r, z, p, q)
            allv = yield from gsum(rr_rz)
            srr = srz = 0.0
            for v in allv:
                srr += v[0]
                srz += v[1]
            iters += 1
            relres = math.sqrt(srr) / gnorm
            relres_prec = math.sqrt(srz if srz > 0.0 else 0.0) / prec0 if prec0 > 0.0 else 0.0
            if relres <= eta:
                reached = True
                break
            beta = srz / rz
            rz = srz
        return iters, relres, relres_prec, reached

    t0 = time.perf_counter()
    rows, stop, message = [], STOP_MAX_ITER, ""

    def row(k, value, gnorm, step, pi, rr, rp):
        x = abi.GnRow()
        x.level, x.iter, x.j_value, x.grad_norm, x.step = level_tag, k, value, gnorm, step
        x.pcg_iters, x.pcg_relres, x.pcg_relres_prec = pi, rr, rp
        x.wall_s = time.perf_counter() - t0
        rows.append(x)

    cur = yield from objective(b, True, grad, None)
    if not cur.feasible:
        raise ValueError("gauss_newton_solve: starting guess is infeasible")
    j_ref = 1.0 + abs((yield from objective(zero, False, None, None)).value)
    _, gg2 = yield from dot(grad, grad)
    grad_norm = math.sqrt(gg2)
    row(0, cur.value, grad_norm, 0.0, 0, 0.0, 0.0)
    if grad_norm <= 1e-15 * j_ref:
        return dict(b=own(b), rows=rows, stop=STOP_CONVERGED,
                    message="gradient numerically zero at start")
    for k in range(1, cfg.max_outer + 1):
        if P.beta > 0.0 and cur.d1max > 1.0 - 1e-10:
            raise ArithmeticError("penalty: derivatives requested at an infeasible point")
        fail = backend.gn_hessian(ext, P, ip_ext, im_ext, b, cfg.precond)
        allv = yield from gsum([float(fail)])
        bad = [int(v[0]) for v in allv if v[0] >= 0]
        if bad:
            raise RuntimeError(f"tridiag factorize: nonpositive pivot in column {min(bad)}")
        piters, prel, prelp, _ = yield from pcg(cfg.eta, cfg.max_pcg)
        gd, _ = yield from dot(grad, dirv)
        if not (gd < 0.0):
            stop, message = STOP_ERROR, "search direction is not a descent direction"
            break
        yield ("halo2", dirv, o0, o1, layer, lo, hi)
        backend.fill0(trial)
        state = {"tev": None, "have": False}

        def phi(t):
            backend.axpy(b, t, dirv, trial)
            ev = yield from objective(trial, True, tgrad, dirv)
            if not ev.feasible:
                return math.inf, 0.0
            state["tev"], state["have"] = ev, True
            return ev.value, ev.dphi

        phi0, dphi0, c1, c2 = cur.value, gd, cfg.wolfe_c1, cfg.wolfe_c2
        evals, lam, ok = 0, 0.0, False
        suff = lambda a, f: f <= phi0 + c1 * a * dphi0  # noqa: E731
        if dphi0 < 0.0 and math.isfinite(phi0):
            prev, lo_p, hi_p = (0.0, phi0, dphi0), None, None
            a, first, zoom = 1.0, True, False
            while evals < cfg.max_ls:
                f, df = yield from phi(a)
                evals += 1
                if not suff(a, f) or (not first and f >= prev[1]):
                    lo_p, hi_p, zoom = prev, (a, f, df), True
                    break
                if abs(df) <= -c2 * dphi0:
                    lam, ok = a, True
                    break
                if df >= 0.0:
                    lo_p, hi_p, zoom = (a, f, df), prev, True
                    break
                prev = (a, f, df)
                a *= 2.0
                first = False
            if zoom:
                while evals < cfg.max_ls:
                    am = 0.5 * (lo_p[0] + hi_p[0])
                    f, df = yield from phi(am)
                    evals += 1
                    if not suff(am, f) or f >= lo_p[1]:
                        hi_p = (am, f, df)
                    else:
                        if abs(df) <= -c2 * dphi0:
                            lam, ok = am, True
                            break
                        if df * (hi_p[0] - lo_p[0]) >= 0.0:
                            hi_p = lo_p
                        lo_p = (am, f, df)
                    if abs(hi_p[0] - lo_p[0]) < 1e-16 * max(1.0, abs(lo_p[0])):
                        break
                if not ok and lo_p[0] > 0.0 and suff(lo_p[0], lo_p[1]):
                    lam, ok = lo_p[0], True
        if not ok:
            stop, message = STOP_LS_FAILURE, "no admissible Wolfe step within the evaluation budget"
            break
        backend.axpy(b, lam, dirv, bnew)
        differs = backend.differs(own(bnew), own(trial))
        allv = yield from gsum([float(differs)])
        tev = state["tev"]
        if not state["have"] or any(v[0] != 0.0 for v in allv):
            tev = yield from objective(bnew, True, tgrad, None)
        _, dd2 = yield from dot(dirv, dirv)
        step_norm = lam * math.sqrt(dd2)
        dj = abs(tev.value - cur.value)
        _, bb2 = yield from dot(b, b)
        bnorm = math.sqrt(bb2)
        _, tg2 = yield from dot(tgrad, tgrad)
        grad_new = math.sqrt(tg2)
        b, bnew = bnew, b
        grad, tgrad = tgrad, grad
        cur, grad_norm = tev, grad_new
        row(k, cur.value, grad_norm, lam, piters, prel, prelp)
        if (dj <= cfg.eps_obj * j_ref and step_norm <= cfg.eps_iter * (1.0 + bnorm)
                and grad_norm <= cfg.eps_grad * j_ref):
            stop = STOP_CONVERGED
            break
    return dict(b=own(b), rows=rows, stop=stop, message=message)


class DeviceGnBackend:
    """GN slab steps on one GPU through the epc_gnslab_* C ABI (torch CUDA
    float64 tensors; see dist_admm.DeviceBackend for the stream rule). The
    GnHessian blocks and the block-Jacobi factor persist in the context
    between epc_gnslab_hessian and the PCG calls, so each rank needs its own
    Context (one per process on a real multi-GPU run)."""

    def __init__(self, ctx, device):
        import torch
        self.ctx, self.lib, self.device, self.torch = ctx, ctx.lib, device, torch

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def fill0(self, x):
        x.zero_()

    def copy(self, dst, src):
        dst.copy_(self.torch.as_tensor(src, device=self.device))

    def view(self, x, first, n):
        return x[first:first + n]

    def differs(self, a, b):
        self._sync()
        return not self.torch.equal(a, b)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def _sync(self):
        self.torch.cuda.synchronize(self.device)

    def _ck(self, rc):
        self.ctx._check(rc)

    def gn_objective(self, ext, P, ip, im, b, need_grad, g_out, d_ext, keep_jac):
        g, k0, mk, lo, hi = ext
        self._sync()
        o = (C.c_double * 8)()
        self._ck(self.lib.epc_gnslab_objective(self.ctx.h, C.byref(g), k0, mk, lo, hi,
                                               self._p(ip), self._p(im), self._p(b), C.byref(P),
                                               int(need_grad), self._p(g_out), self._p(d_ext),
                                               int(keep_jac), o))
        return list(o)

    def gn_hessian(self, ext, P, ip, im, b, kind):
        g, k0, mk, lo, hi = ext
        self._sync()
        f = C.c_longlong(-1)
        self._ck(self.lib.epc_gnslab_hessian(self.ctx.h, C.byref(g), k0, mk, lo, hi, self._p(ip),
                                             self._p(im), self._p(b), C.byref(P), kind,
                                             C.byref(f)))
        return f.value

    def gn_hv(self, ext, P, p, q):
        g, k0, mk, lo, hi = ext
        self._sync()
        o = C.c_double()
        self._ck(self.lib.epc_gnslab_hv(self.ctx.h, C.byref(g), k0, mk, lo, hi, C.byref(P),
                                        self._p(p), self._p(q), C.byref(o)))
        return o.value

    def gn_update(self, ext, P, kind, a, do_axpy, d, r, z, p, q):
        g, k0, mk, lo, hi = ext
        self._sync()
        o = (C.c_double * 2)()
        self._ck(self.lib.epc_gnslab_update(self.ctx.h, C.byref(g), k0, mk, lo, hi, C.byref(P),
                                            kind, a, int(do_axpy), self._p(d), self._p(r),
                                            self._p(z), self._p(p), self._p(q), o))
        return list(o)

    def axpy(self, x, t, d, y):
        self._sync()
        self._ck(self.lib.epc_gnslab_axpy(self.ctx.h, y.numel(), self._p(x), t, self._p(d),
                                          self._p(y)))

    def negate(self, g, r):
        self._sync()
        o = C.c_double()
        self._ck(self.lib.epc_gnslab_negate(self.ctx.h, g.numel(), self._p(g), self._p(r),
                                            C.byref(o)))
        return o.value

    def dot(self, a, b):
        self._sync()
        o = (C.c_double * 2)()
        self._ck(self.lib.epc_gnslab_dot(self.ctx.h, a.numel(), self._p(a), self._p(b), o))
        return list(o)
