"""Slab-distributed ADMM: one volume over several GPUs.

The volume is split into k-slabs (internal axis 3, shard_range over m3):
rank r owns face layers [k0, k0 + mk). One iteration of admm_solve
(proj/src/admm.cpp:488-560) becomes, per rank:

  b-step on the slab's columns (columns (j, k) never couple)    local
  z-step: rho V (b + u), axis-2 DCT, pack rank blocks          local
          all-to-all  k-slabs -> i-slabs                        exchange
          axis-3 DCT, spectral divide, inverse axis-3 DCT       local
          all-to-all  i-slabs -> k-slabs                        exchange
          inverse axis-2 DCT, u += b - z, residual sums         local
  g(z): one face layer of z from rank r+1 (the D3 boundary)     halo
  all-gather of ~15 scalars; rows, stop test, rho schedule      replicated

Every rank runs the same generator (`admm_rank`): it yields its collective
requests and receives their results, so the same code runs
  * under torch.distributed (`run_torch`: NCCL on GPUs, gloo on CPU), and
  * as G ranks in lockstep inside one process (`run_lockstep`) - the
    single-GPU check of the decomposition (each rank's kernels run in turn;
    no rank ever waits on another's kernels).
The local steps are a backend: `DeviceBackend` drives the C ABI slab entry
points (epc_slab_*, csrc/slab_host.inc) on torch CUDA tensors; the CPU tests
plug in a backend built on the oracle. Scalars are reduced in rank order on
every rank, so the replicated decisions are identical and deterministic.
With one rank the iteration is the single-GPU epc_admm_solve's (bitwise).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

from . import abi, decide, shard

STOP_CONVERGED, STOP_MAX_ITER, STOP_ERROR = 0, 1, 3  # EPC_STOP_* (include/epicorr_b200.h)
QP_WHAT = {1: "column factor: nonpositive pivot",
           2: "qp_active_set: infeasible starting point",
           3: "qp_active_set: singular Schur complement",
           4: "qp_active_set: iteration cap reached (cycling guard)"}


@dataclass(frozen=True)
class Slabs:
    """k-slab ownership (faces layout i + n1 (j + m2 k)) and the i-slab
    ownership used during the axis-3 transform, both by shard_range."""
    m1: int
    m2: int
    m3: int
    world: int

    @property
    def n1(self):
        return self.m1 + 1

    def k_range(self, r):
        return shard.shard_range(self.m3, r, self.world)

    def i_range(self, s):
        return shard.shard_range(self.n1, s, self.world)

    def slab_faces(self, r):
        return self.n1 * self.m2 * self.k_range(r)[1]

    def slab_cells(self, r):
        return self.m1 * self.m2 * self.k_range(r)[1]

    def islab_faces(self, s):
        return self.i_range(s)[1] * self.m2 * self.m3

    def block(self, sender, receiver):
        """Elements sender -> receiver in the forward transpose."""
        return self.i_range(receiver)[1] * self.m2 * self.k_range(sender)[1]


def rho_schedule(schedule, rho, rho_min, pr, du, ti, td, mu):
    """admm.cpp:478-486 (the same arithmetic as api.cu's rho_schedule)."""
    if schedule == abi.RHO_FIXED:
        return rho
    nxt = rho
    if pr > mu * du:
        nxt = rho * ti
    elif du > mu * pr:
        nxt = rho / td
    if schedule == abi.RHO_ADAPTIVE_BOUNDED:
        nxt = rho_min if nxt < rho_min else nxt  # std::max(next, rho_min)
    return nxt


def admm_rank(backend, grid, slabs, rank, ip, im, cfg=None, params=None, rho0=None, level_tag=0,
              state=None, exact_sums=False):
    """One rank of the distributed admm_solve (a generator; see module doc).
    ip / im: this rank's cell slab; state: optional (b, z, u) face slabs.
    exact_sums: take every stop / rho decision on the reference's sequential
    sums (EPC_MODE_EXACT_SUMS), not only the undecidable ones.
    Returns dict(b, z, u, rho, rows, stop, message, decisions) for the rank's
    slab; decisions = [certified, exact]."""
    cfg = cfg or abi.AdmmConfig()
    params = params or abi.ObjectiveParams()
    world = slabs.world
    k0, mk = slabs.k_range(rank)
    i0, ni = slabs.i_range(rank)
    nf = slabs.slab_faces(rank)
    layer = slabs.n1 * slabs.m2
    V = grid.h[0] * grid.h[1] * grid.h[2]
    sqrt_n = math.sqrt(float(slabs.n1 * slabs.m2 * slabs.m3))
    B = [backend.zeros(nf), backend.zeros(nf)]
    Z = [backend.zeros(nf), backend.zeros(nf)]
    U = [backend.zeros(nf), backend.zeros(nf)]
    if state is not None:
        for dst, src in zip((B[0], Z[0], U[0]), state):
            if src is not None:
                backend.copy(dst, src)
    send_f = backend.zeros(nf)                      # rank blocks (forward)
    isl_in = backend.zeros(slabs.islab_faces(rank))  # i-slab received
    isl_out = backend.zeros(slabs.islab_faces(rank))
    recv_b = backend.zeros(nf)                      # rank blocks (return)
    fwd_send = [slabs.block(rank, s) for s in range(world)]
    fwd_recv = [slabs.block(s, rank) for s in range(world)]
    if state is not None and state[0] is not None:
        # admm.cpp:501-502: norm_inf(diff_x1(b)) > 1 throws before iteration 1
        allm = yield ("gather", [backend.d1_norm_inf(grid, k0, mk, B[0])])
        if max(v[0] for v in allm) > 1.0:
            raise ValueError("admm_solve: infeasible starting field")
    rho = rho0 if (rho0 is not None and rho0 > 0.0) else cfg.rho0
    rows, stop, message = [], STOP_MAX_ITER, ""
    ndec = [0, 0]
    adaptive = cfg.schedule != abi.RHO_FIXED
    nface_total = slabs.n1 * slabs.m2 * slabs.m3
    t0 = time.perf_counter()
    for it in range(1, cfg.max_iter + 1):
        tb = time.perf_counter()
        sums3, ints4 = backend.bstep(grid, k0, mk, ip, im, B[0], Z[0], U[0], rho, params, cfg,
                                     B[1])
        tb = time.perf_counter() - tb
        backend.zforward(grid, k0, mk, world, B[1], U[0], rho, send_f)
        yield ("alltoall", send_f, fwd_send, isl_in, fwd_recv)
        backend.zsolve3(grid, ni, isl_in, params.alpha, rho, isl_out)
        yield ("alltoall", isl_out, fwd_recv, recv_b, fwd_send)
        sums6 = backend.zbackward(grid, k0, mk, world, recv_b, B[1], U[0], Z[0], rho, Z[1], U[1])
        halo = yield ("halo_up", backend.view(Z[1], 0, layer))
        sums2 = backend.zdiff(grid, k0, mk, Z[1], halo)
        mine = [sums3[0], sums3[1], sums3[2], float(ints4[0]), float(ints4[1]), float(ints4[2]),
                float(ints4[3])] + list(sums6) + list(sums2) + [tb]
        allv = yield ("gather", mine)
        # ---- replicated reduction, rank order ------------------------------
        kkt = fr = fd = 0.0
        du = [0.0] * 6
        zd = [0.0, 0.0]
        err_col, err_code, bsec = -1, 0, 0.0
        for v in allv:
            kkt = v[0] if kkt < v[0] else kkt
            fr += v[1]
            fd += v[2]
            if v[3] >= 0 and (err_col < 0 or v[3] < err_col):
                err_col, err_code = int(v[3]), int(v[4])
            for q in range(6):
                du[q] += v[7 + q]
            zd[0] += v[13]
            zd[1] += v[14]
            bsec = max(bsec, v[15])
        if err_col >= 0:  # admm.cpp:553-557: stop = error, state from before
            stop = STOP_ERROR
            message = f"b_update: column {err_col}: {QP_WHAT.get(err_code, 'unknown column failure')}"
            break
        row = abi.AdmmRow()
        row.level, row.iter, row.rho, row.kkt_violation = level_tag, it, rho, kkt
        row.b_update_s = bsec
        row.primal_res, row.dual_res, row.eps_pri, row.eps_dual = decide.residuals(
            du, rho, V, sqrt_n, cfg.eps_abs, cfg.eps_rel)
        # stop test and rho schedule (admm.cpp:542-548), certified against the
        # reference's sequential sums (decide.py); undecidable -> the exact
        # chains, continued rank after rank in index order
        dec = None if exact_sums else decide.certified(du, nface_total, rho, V, sqrt_n, cfg.eps_abs,
                                                       cfg.eps_rel, cfg.mu, adaptive)
        if dec is not None:
            ndec[0] += 1
        else:
            seq = [0.0] * 5
            for r in range(world):
                if r == rank:
                    seq = backend.seq_sums(B[1], Z[1], Z[0], U[1], seq)
                seq = yield ("bcast", list(seq), r)
            row.primal_res, row.dual_res, row.eps_pri, row.eps_dual = decide.residuals(
                seq, rho, V, sqrt_n, cfg.eps_abs, cfg.eps_rel)
            dec = decide.exact(seq, rho, V, sqrt_n, cfg.eps_abs, cfg.eps_rel, cfg.mu, adaptive)
            ndec[1] += 1
        fval = 0.5 * V * fr + 0.5 * params.alpha * V * fd
        gs = zd[0] + (zd[1] if grid.dim == 3 else 0.0)
        gval = 0.5 * params.alpha * V * gs
        row.lagrangian = fval + gval + rho * V * du[5] + 0.5 * rho * V * du[0]
        row.wall_s = time.perf_counter() - t0
        rows.append(row)
        B.reverse()
        Z.reverse()
        U.reverse()
        if dec[0]:
            stop = STOP_CONVERGED
            break
        nxt = decide.rho_apply(cfg.schedule, rho, cfg.rho_min, dec[1], cfg.tau_incr, cfg.tau_decr,
                               abi.RHO_FIXED, abi.RHO_ADAPTIVE_BOUNDED)
        if nxt != rho:
            backend.scale(U[0], rho / nxt)
            rho = nxt
    return dict(b=B[0], z=Z[0], u=U[0], rho=rho, rows=rows, stop=stop, message=message,
                decisions=ndec)


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------
def run_lockstep(gens, cat, split):
    """Run G rank generators in one process, performing their collectives
    in memory. cat(list) concatenates buffers; split(buf, counts) splits."""
    world = len(gens)
    reqs = [next(g) for g in gens]
    results = [None] * world
    while True:
        kind = reqs[0][0]
        assert all(r[0] == kind for r in reqs), "ranks diverged"
        if kind == "alltoall":
            parts = [split(r[1], r[2]) for r in reqs]  # parts[sender][receiver]
            answers = []
            for dst in range(world):
                buf = reqs[dst][3]
                got = cat([parts[s][dst] for s in range(world)])
                buf[:] = got
                answers.append(buf)
        elif kind == "halo_up":
            answers = [reqs[r + 1][1] if r + 1 < world else None for r in range(world)]
        elif kind == "halo2":
            # ("halo2", x_ext, o0, o1, layer, lo, hi): first owned layer -> the
            # lower rank's upper halo, last owned layer -> the upper rank's
            # lower halo (in place)
            for r in range(world):
                x, o0, o1, lay = reqs[r][1], reqs[r][2], reqs[r][3], reqs[r][4]
                if r > 0:
                    y, yo1 = reqs[r - 1][1], reqs[r - 1][3]
                    y[yo1:yo1 + lay] = x[o0:o0 + lay]
                if r + 1 < world:
                    reqs[r + 1][1][0:lay] = x[o1 - lay:o1]
            answers = [None] * world
        elif kind == "gather":
            vals = [list(r[1]) for r in reqs]
            answers = [vals] * world
        elif kind == "bcast":
            root = reqs[0][2]
            answers = [list(reqs[root][1])] * world
        else:
            raise RuntimeError(kind)
        nxt = []
        done = 0
        for r, g in enumerate(gens):
            try:
                nxt.append(g.send(answers[r]))
            except StopIteration as e:
                results[r] = e.value
                done += 1
                nxt.append(None)
        if done:
            assert done == world, "ranks finished at different iterations"
            return results
        reqs = nxt


def run_torch(gen, dist, device, timings=None):
    """Run this rank's generator with torch.distributed collectives
    (NCCL for CUDA tensors, gloo for CPU tensors). timings: optional dict,
    accumulates seconds and counts per collective kind (each collective is
    then bracketed by device synchronisations)."""
    import time as _time

    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    as_t = _as_tensor
    cuda = isinstance(device, torch.device) and device.type == "cuda"
    try:
        req = next(gen)
        while True:
            kind = req[0]
            if timings is not None:
                if cuda:
                    torch.cuda.synchronize(device)
                t_req = _time.perf_counter()
            if kind == "alltoall":
                _, send, scounts, recv, rcounts = req
                ts, tr = as_t(send), as_t(recv)
                dist.all_to_all_single(tr, ts, output_split_sizes=list(rcounts),
                                       input_split_sizes=list(scounts))
                ans = recv
            elif kind == "halo_up":
                mine = as_t(req[1]).contiguous()
                got = torch.empty_like(mine) if rank + 1 < world else None
                ops = []
                if rank > 0:
                    ops.append(dist.P2POp(dist.isend, mine, rank - 1))
                if got is not None:
                    ops.append(dist.P2POp(dist.irecv, got, rank + 1))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                ans = None if got is None else _like(req[1], got)
            elif kind == "halo2":
                _, x, o0, o1, lay, lo, hi = req
                tx = as_t(x)
                ops = []
                if lo:   # rank - 1 exists: its halo <- my first layer, mine <- its last
                    ops.append(dist.P2POp(dist.isend, tx[o0:o0 + lay].contiguous(), rank - 1))
                    lo_buf = torch.empty_like(tx[0:lay])
                    ops.append(dist.P2POp(dist.irecv, lo_buf, rank - 1))
                if hi:
                    ops.append(dist.P2POp(dist.isend, tx[o1 - lay:o1].contiguous(), rank + 1))
                    hi_buf = torch.empty_like(tx[0:lay])
                    ops.append(dist.P2POp(dist.irecv, hi_buf, rank + 1))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                if lo:
                    tx[0:lay].copy_(lo_buf)
                if hi:
                    tx[o1:o1 + lay].copy_(hi_buf)
                ans = None
            elif kind == "gather":
                t = torch.tensor(req[1], dtype=torch.float64, device=device)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t)
                ans = [o.cpu().tolist() for o in outs]
            elif kind == "bcast":
                t = torch.tensor(req[1], dtype=torch.float64, device=device)
                dist.broadcast(t, src=req[2])
                ans = t.cpu().tolist()
            else:
                raise RuntimeError(kind)
            if timings is not None:
                if cuda:
                    torch.cuda.synchronize(device)
                tk = timings.setdefault(kind, [0.0, 0])
                tk[0] += _time.perf_counter() - t_req
                tk[1] += 1
            req = gen.send(ans)
    except StopIteration as e:
        return e.value


def _as_tensor(x):
    import numpy as np
    import torch
    if isinstance(x, np.ndarray):
        return torch.from_numpy(x)
    return x


def _like(proto, t):
    import numpy as np
    if isinstance(proto, np.ndarray):
        return t.numpy()
    return t


# ---------------------------------------------------------------------------
# device backend (the product): C ABI slab steps on torch CUDA tensors
# ---------------------------------------------------------------------------
class DeviceBackend:
    """Local steps on one GPU through the epc_slab_* C ABI. Buffers are
    torch float64 CUDA tensors; the context's stream is used for the
    kernels, torch's current stream for the collectives (synchronised at
    each step boundary by the ABI's scalar read-backs)."""

    def __init__(self, ctx, device):
        import torch
        self.ctx, self.lib, self.device = ctx, ctx.lib, device
        self.torch = torch

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def copy(self, dst, src):
        dst.copy_(self.torch.as_tensor(src, device=self.device))

    def view(self, x, first, n):
        return x[first:first + n]

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def _sync_torch(self):
        # kernels run on the context stream; make torch's stream (used by
        # the collectives) wait for them
        self.torch.cuda.synchronize(self.device)

    def bstep(self, g, k0, mk, ip, im, b, z, u, rho, params, cfg, b_out):
        self._sync_torch()  # inputs may have been produced on any torch stream
        s3 = (C.c_double * 3)()
        i4 = (C.c_longlong * 4)()
        self.ctx._check(self.lib.epc_slab_bstep(self.ctx.h, C.byref(g), k0, mk, self._p(ip),
                                                self._p(im), self._p(b), self._p(z), self._p(u),
                                                rho, C.byref(params), C.byref(cfg), self._p(b_out),
                                                s3, i4))
        return list(s3), list(i4)

    def zforward(self, g, k0, mk, world, b, u, rho, blocks):
        self.ctx._check(self.lib.epc_slab_zforward(self.ctx.h, C.byref(g), k0, mk, world,
                                                   self._p(b), self._p(u), rho, self._p(blocks)))
        self._sync_torch()

    def zsolve3(self, g, ni, inp, alpha, rho, out):
        self._sync_torch()
        self.ctx._check(self.lib.epc_slab_zsolve3(self.ctx.h, C.byref(g), ni, self._p(inp), alpha,
                                                  rho, self._p(out)))
        self._sync_torch()

    def zbackward(self, g, k0, mk, world, blocks, b, u_old, z_old, rho, z_new, u_new):
        self._sync_torch()
        s6 = (C.c_double * 6)()
        self.ctx._check(self.lib.epc_slab_zbackward(self.ctx.h, C.byref(g), k0, mk, world,
                                                    self._p(blocks), self._p(b), self._p(u_old),
                                                    self._p(z_old), rho, self._p(z_new),
                                                    self._p(u_new), s6))
        return list(s6)

    def zdiff(self, g, k0, mk, z, halo):
        self._sync_torch()
        s2 = (C.c_double * 2)()
        self.ctx._check(self.lib.epc_slab_zdiff(self.ctx.h, C.byref(g), k0, mk, self._p(z),
                                                self._p(halo), s2))
        return list(s2)

    def seq_sums(self, b_new, z_new, z_old, u_new, start):
        self._sync_torch()
        io = (C.c_double * 5)(*start)
        self.ctx._check(self.lib.epc_slab_seq_sums(self.ctx.h, b_new.numel(), self._p(b_new),
                                                   self._p(z_new), self._p(z_old), self._p(u_new),
                                                   io))
        return list(io)

    def d1_norm_inf(self, g, k0, mk, b):
        self._sync_torch()
        out = C.c_double(0.0)
        self.ctx._check(self.lib.epc_slab_d1_norm_inf(self.ctx.h, C.byref(g), k0, mk, self._p(b),
                                                      C.byref(out)))
        return out.value

    def scale(self, x, factor):
        self.ctx._check(self.lib.epc_slab_scale(self.ctx.h, x.numel(), self._p(x), factor))
        self._sync_torch()


def torch_cat(parts):
    import torch
    return torch.cat(parts)


def torch_split(buf, counts):
    return list(buf.split(list(counts)))
