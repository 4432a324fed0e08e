"""CPU backend of the slab-distributed ADMM (paper_1607_00531_b200/dist_admm.py)
for tests: the b-step through the oracle (the C restatement, bitwise pinned to
the reference) on the slab's columns, the DCT pieces as exact-k-order numpy
products with the reference's matrices (dct2_matrix / neumann_eigenvalues,
operators.cpp:275-295, evaluated with the C library's cos/sin like the C++
host code). Test infrastructure only - the product path is DeviceBackend."""
import math

import numpy as np

from paper_1607_00531_b200 import abi

PI = 3.141592653589793238462643383279502884


def dct2_matrix(m):
    s0, sq = math.sqrt(1.0 / m), math.sqrt(2.0 / m)
    c = np.empty((m, m))
    for q in range(m):
        for j in range(m):
            c[q, j] = (s0 if q == 0 else sq) * math.cos(PI * q * (2.0 * j + 1.0) / (2.0 * m))
    return c


def neumann_eigenvalues(m, h):
    lam = np.empty(m)
    for q in range(m):
        s = math.sin(PI * q / (2.0 * m))
        lam[q] = 4.0 / (h * h) * s * s
    return lam


def ordered_apply(A, X, axis):
    """out[q] = sum_k A[q, k] X[k] along `axis`, k ascending from 0, separate
    multiply and add (the reference's transform loops)."""
    X = np.moveaxis(X, axis, 0)
    acc = np.zeros((A.shape[0],) + X.shape[1:])
    for k in range(A.shape[1]):
        acc = acc + A[:, k].reshape((-1,) + (1,) * (X.ndim - 1)) * X[k][None]
    return np.moveaxis(acc, 0, axis)


class OracleBackend:
    def __init__(self, oracle, grid):
        self.orc, self.g = oracle, grid
        m1, m2, m3 = grid.m
        self.c2, self.c3 = dct2_matrix(m2), dct2_matrix(m3)
        self.l2, self.l3 = neumann_eigenvalues(m2, grid.h[1]), neumann_eigenvalues(m3, grid.h[2])
        self.V = grid.h[0] * grid.h[1] * grid.h[2]

    def _slab_grid(self, mk):
        g = self.g
        return abi.Grid.make(g.m[0], g.m[1], mk, h=tuple(g.h), origin=tuple(g.origin), dim=3)

    def zeros(self, n):
        return np.zeros(n)

    def copy(self, dst, src):
        dst[:] = src

    def view(self, x, first, n):
        return x[first:first + n]

    def seq_sums(self, b_new, z_new, z_old, u_new, start):
        """The reference's sequential chains (np.add.accumulate adds in index
        order, one rounding per element), continued from start."""
        terms = [(b_new - z_new) ** 2, (z_old - z_new) ** 2, b_new * b_new, z_new * z_new,
                 u_new * u_new]
        return [float(np.add.accumulate(np.concatenate(([s0], t)))[-1]) for s0, t in zip(start, terms)]

    def d1_norm_inf(self, g, k0, mk, b):
        bb = b.reshape(-1, g.m[0] + 1)
        return float(np.abs((bb[:, 1:] - bb[:, :-1]) * (1.0 / g.h[0])).max())  # diff_x1, operators.cpp:45-49

    def bstep(self, g, k0, mk, ip, im, b, z, u, rho, params, cfg, b_out):
        sg = self._slab_grid(mk)
        r = self.orc.b_update(sg, ip, im, b, z, u, rho, params=params, cfg=cfg)
        if r["rc"] != 0:
            raise RuntimeError(r["message"])
        b_out[:] = r["b"]
        res = self.orc.residual(sg, ip, im, b_out)
        bb = b_out.reshape(-1, sg.n1)
        d = (bb[:, 1:] - bb[:, :-1]) * (1.0 / g.h[0])
        return ([r["kkt_violation"], float(np.sum(res * res)), float(np.sum(d * d))],
                [-1, 0, r["sqp_iters"], r["qp_iters"]])

    def zforward(self, g, k0, mk, world, b, u, rho, blocks):
        m1, m2, _ = g.m
        n1 = m1 + 1
        wrhs = rho * self.V
        rhs = (wrhs * (b + u)).reshape(mk, m2, n1)
        h = ordered_apply(self.c2, rhs, 1)
        parts = []
        for s in range(world):
            i0, ni = _split(n1, s, world)
            parts.append(h[:, :, i0:i0 + ni].reshape(-1))
        blocks[:] = np.concatenate(parts)

    def zsolve3(self, g, ni, inp, alpha, rho, out):
        m1, m2, m3 = g.m
        X = inp.reshape(m3, m2, ni)
        H = ordered_apply(self.c3, X, 0)
        lam = self.l2[None, :] + self.l3[:, None]          # [q3][j]
        den = alpha * self.V * lam + rho * self.V
        H = H / den[:, :, None]
        out[:] = ordered_apply(self.c3.T, H, 0).reshape(-1)

    def zbackward(self, g, k0, mk, world, blocks, b, u_old, z_old, rho, z_new, u_new):
        m1, m2, _ = g.m
        n1 = m1 + 1
        h = np.empty((mk, m2, n1))
        off = 0
        for s in range(world):
            i0, ni = _split(n1, s, world)
            cnt = mk * m2 * ni
            h[:, :, i0:i0 + ni] = blocks[off:off + cnt].reshape(mk, m2, ni)
            off += cnt
        z = ordered_apply(self.c2.T, h, 1).reshape(-1)
        z_new[:] = z
        diff = b - z
        un = u_old + diff
        u_new[:] = un
        dz = z_old - z
        return [float(np.sum(diff * diff)), float(np.sum(dz * dz)), float(np.sum(b * b)),
                float(np.sum(z * z)), float(np.sum(un * un)), float(np.sum(un * diff))]

    def zdiff(self, g, k0, mk, z, halo):
        m1, m2, _ = g.m
        n1 = m1 + 1
        Z = z.reshape(mk, m2, n1)
        d2 = (Z[:, 1:, :] - Z[:, :-1, :]) * (1.0 / g.h[1])
        d3 = (Z[1:] - Z[:-1]) * (1.0 / g.h[2])
        s3 = float(np.sum(d3 * d3))
        if halo is not None:
            e = (halo.reshape(m2, n1) - Z[-1]) * (1.0 / g.h[2])
            s3 += float(np.sum(e * e))
        return [float(np.sum(d2 * d2)), s3]

    def scale(self, x, factor):
        if factor != 1.0:
            x *= factor


def _split(n, s, world):
    base, extra = divmod(n, world)
    return s * base + min(s, extra), base + (1 if s < extra else 0)


def np_cat(parts):
    return np.concatenate(parts)


def np_split(buf, counts):
    out, o = [], 0
    for c in counts:
        out.append(buf[o:o + c])
        o += c
    return out
