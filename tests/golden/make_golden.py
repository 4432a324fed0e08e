"""Generate tests/golden/*.npz from the REFERENCE library (oracle/_ref, the
unmodified proj/src compiled by oracle/Makefile). Run in the container that
has /root/reference; the fixtures are committed so the GPU box (no
reference tree) can check the oracle and the product against them.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ffi  # noqa: E402
from paper_1607_00531_b200 import abi, synth  # noqa: E402

EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


def grid_arr(g):
    return np.array([g.dim, *g.m, *g.h, *g.origin], dtype=np.float64)


def rows_arr(rows, keys):
    return np.array([[r[k] for k in keys] for r in rows], dtype=np.float64)


ADMM_KEYS = ["iter", "primal_res", "dual_res", "eps_pri", "eps_dual", "rho", "lagrangian",
             "kkt_violation"]
GN_KEYS = ["iter", "j_value", "grad_norm", "step", "pcg_iters", "pcg_relres", "pcg_relres_prec"]


def main():
    ref = ffi.load("ref")
    out = {}
    # ADMM solves (3D anisotropic-free synthetic pairs, both intensity scales)
    for name, m, seed, scale, iters in (("admm_a", (16, 12, 8), 7, 1.0, 20),
                                        ("admm_b", (16, 12, 8), 7, 400.0, 20),
                                        ("admm_c", (24, 20, 1), 3, 400.0, 15)):
        d = synth.make_pair(synth.SynthSpec(m=m, seed=seed))
        g = d.grid if m[2] > 1 else abi.Grid.make(m[0], m[1], 1)
        ip, im = d.iplus * scale, d.iminus * scale
        r = ref.admm_solve(g, ip, im, cfg=abi.AdmmConfig(max_iter=iters, **EXACT))
        out[name] = dict(grid=grid_arr(g), iplus=ip, iminus=im, b=r["b"], z=r["z"], u=r["u"],
                         rho=np.array([r["rho"]]), stop=np.array([r["stop"]]),
                         rows=rows_arr(r["rows"], ADMM_KEYS), max_iter=np.array([iters]))
    # GN solves
    for name, m, seed, scale in (("gn_a", (20, 16, 10), 9, 1.0), ("gn_b", (20, 16, 10), 9, 400.0)):
        d = synth.make_pair(synth.SynthSpec(m=m, seed=seed))
        ip, im = d.iplus * scale, d.iminus * scale
        cfg = abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=10)
        r = ref.gn_solve(d.grid, ip, im, cfg=cfg)
        out[name] = dict(grid=grid_arr(d.grid), iplus=ip, iminus=im, b=r["b"],
                         stop=np.array([r["stop"]]), rows=rows_arr(r["rows"], GN_KEYS))
    # column QPs (test_admm.cpp:126-147 style: 5 faces, h = 0.8, seeded)
    rng = np.random.default_rng(77)
    n, h, nq = 5, 0.8, 200
    gd = 2.5 + rng.uniform(-1, 1, (nq, n))
    go = np.zeros((nq, n))
    go[:, :-1] = 0.9 * rng.uniform(-1, 1, (nq, n - 1))
    c = 4.0 * rng.uniform(-1, 1, (nq, n))
    xs, lams, signs, its = [], [], [], []
    for q in range(nq):
        r = ref.qp_active_set(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), np.zeros(n), 200)
        xs.append(r["x"])
        lams.append(r["lam"])
        signs.append(r["sign"])
        its.append(r["iters"])
    out["qp5"] = dict(gd=gd, go=go, c=c, h=np.array([h]), x=np.array(xs), lam=np.array(lams),
                      sign=np.array(signs), iters=np.array(its))
    # z-update on an anisotropic 3D grid (test_admm.cpp:260-296 shape)
    g = abi.Grid.make(6, 5, 4, h=(0.5, 1.0, 1.5))
    rng = np.random.default_rng(79)
    b, u = rng.uniform(-1, 1, g.faces), rng.uniform(-1, 1, g.faces)
    out["zupd"] = dict(grid=grid_arr(g), b=b, u=u, z=ref.z_update(g, b, u, 3.0, 7.0))
    for name, arrs in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrs)
        print(name, {k: v.shape for k, v in arrs.items()})


if __name__ == "__main__":
    main()
