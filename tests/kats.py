"""Known-answer checks restated from the reference's own unit tests
(proj/tests/test_admm.cpp, test_operators.cpp, test_gn_pcg.cpp,
test_objective.cpp). Each takes an implementation `impl` exposing the
shared method names (the CPU oracle or the GPU Context) and asserts the
reference's expected values. Collected by test_kats_oracle.py (CPU) and
test_gpu_kats.py (GPU)."""
import itertools

import numpy as np

from paper_1607_00531_b200 import abi, synth

APPROX = dict(rel=1e-12)


def _close(a, b, rel=1e-12, abs_=0.0):
    return abs(a - b) <= max(rel * abs(b), abs_)


def brute_force_qp(n, h, gd, go, c):
    """Exhaustive 3^k active-set enumeration (test_admm.cpp:19-93): solve the
    bordered KKT system per sign pattern, keep the feasible, dual-feasible
    candidate with the lowest objective."""
    G = np.diag(gd) + np.diag(go[:-1], 1) + np.diag(go[:-1], -1)
    best, best_x = np.inf, None
    for signs in itertools.product((0, 1, -1), repeat=n - 1):
        act = [(i, s) for i, s in enumerate(signs) if s != 0]
        na = len(act)
        K = np.zeros((n + na, n + na))
        rhs = np.zeros(n + na)
        K[:n, :n] = G
        rhs[:n] = -c
        for r, (i, s) in enumerate(act):
            a = s / h
            K[n + r, i], K[n + r, i + 1] = -a, a
            K[i, n + r], K[i + 1, n + r] = -a, a
            rhs[n + r] = -1.0
        try:
            sol = np.linalg.solve(K, rhs)
        except np.linalg.LinAlgError:
            continue
        if any(-sol[n + r] < -1e-9 for r in range(na)):
            continue
        x = sol[:n]
        if np.any(np.abs(np.diff(x) / h) > 1 + 1e-9):
            continue
        obj = 0.5 * x @ G @ x + c @ x
        if obj < best - 1e-12:
            best, best_x = obj, x
    return best_x


def qp_batch(impl, n, h, gd, go, c, x0, cap):
    """Uniform QP call: GPU Context has a batched entry point, the oracle a
    per-QP one."""
    gd, go, c, x0 = (np.atleast_2d(np.asarray(a, dtype=np.float64)) for a in (gd, go, c, x0))
    if hasattr(impl, "qp_active_set_batch"):
        r = impl.qp_active_set_batch(n, h, gd, go, c, x0, cap)
        return [dict(x=r["x"][q], lam=r["lam"][q], sign=r["sign"][q], rc=int(r["status"][q]),
                     kkt=r["kkt"][q], message=r["message"]) for q in range(gd.shape[0])]
    out = []
    for q in range(gd.shape[0]):
        r = impl.qp_active_set(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), x0[q].copy(), cap)
        kkt = impl.verify_qp_kkt(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), r["x"], r["lam"],
                                 r["sign"]) if r["rc"] == 0 else np.nan
        out.append(dict(x=r["x"], lam=r["lam"], sign=r["sign"], rc=r["rc"], kkt=kkt,
                        message=r["message"]))
    return out


def kat_qp_two_face(impl):
    # test_admm.cpp:101-124
    r = qp_batch(impl, 2, 1.0, [1, 1], [0, 0], [0, 0], [0, 0], 50)[0]
    assert r["rc"] == 0 and not r["x"].any() and r["sign"][0] == 0 and r["lam"][0] == 0.0
    r = qp_batch(impl, 2, 1.0, [1, 1], [0, 0], [-3, 3], [0, 0], 50)[0]
    assert _close(r["x"][0], 0.5) and _close(r["x"][1], -0.5)
    assert r["sign"][0] == 1 and _close(r["lam"][0], 2.5) and r["kkt"] <= 1e-10
    r = qp_batch(impl, 2, 1.0, [1, 1], [0, 0], [0, 0], [0, 5.0], 50)[0]
    assert r["rc"] == abi.EPC_ERR_INVALID_ARGUMENT


def kat_qp_cycling_guard(impl):
    # test_admm.cpp:149-153
    r = qp_batch(impl, 3, 1.0, [1, 1, 1], [0, 0, 0], [-9, 0, 9], [0, 0, 0], 1)[0]
    assert r["rc"] == abi.EPC_ERR_RUNTIME and "cycling guard" in r["message"]


def kat_qp_brute_force(impl, trials=200):
    # test_admm.cpp:126-147: 200 random 5-face QPs vs exhaustive enumeration
    rng = np.random.default_rng(77)
    n, h = 5, 0.8
    gd = 2.5 + rng.uniform(-1, 1, (trials, n))
    go = np.zeros((trials, n))
    go[:, :-1] = 0.9 * rng.uniform(-1, 1, (trials, n - 1))
    c = 4.0 * rng.uniform(-1, 1, (trials, n))
    res = qp_batch(impl, n, h, gd, go, c, np.zeros((trials, n)), 200)
    for q in range(trials):
        expect = brute_force_qp(n, h, gd[q], go[q], c[q])
        assert expect is not None
        r = res[q]
        assert r["rc"] == 0
        assert np.allclose(r["x"], expect, rtol=1e-7, atol=1e-9)
        assert r["kkt"] <= 1e-8
        assert np.all(np.abs(np.diff(r["x"]) / h) <= 1.0 + 1e-12)


def kat_dual_update(impl):
    # test_admm.cpp:298-322: n = 100 faces (4x20 cells)
    g = abi.Grid.make(4, 20, 1)
    assert g.faces == 100
    b, z, zo, u = (np.zeros(100) for _ in range(4))
    b[0], z[0] = 5.0, 1.0
    un, r = impl.dual_update(g, b, z, zo, u, 2.0, 0.2, 0.2)
    assert _close(r["eps_pri"], np.sqrt(100.0) * 0.2 + 0.2 * 5.0, 1e-15)
    assert _close(r["eps_pri"], 3.0, 1e-15)
    assert _close(r["primal_res"], 4.0, 1e-15)
    assert _close(un[0], 4.0, 1e-15)
    same = np.zeros(100)
    same[3] = 2.0
    un2, r2 = impl.dual_update(g, same, same, same, u, 2.0, 0.2, 0.2)
    assert r2["primal_res"] == 0.0 and np.array_equal(un2, u)
    _, r3 = impl.dual_update(g, b, z, z, u, 2.0, 0.2, 0.2)
    assert r3["dual_res"] == 0.0


def kat_rho_schedule(impl):
    # test_admm.cpp:324-331
    f, a, ab = abi.RHO_FIXED, abi.RHO_ADAPTIVE, abi.RHO_ADAPTIVE_BOUNDED
    assert impl.rho_schedule(f, 7.0, 1.0, 100.0, 1.0, 2, 2, 10) == 7.0
    assert impl.rho_schedule(a, 8.0, 1.0, 5.0, 5.0, 2, 2, 10) == 8.0
    assert impl.rho_schedule(a, 8.0, 1.0, 20.0, 1.0, 2, 2, 10) == 16.0
    assert impl.rho_schedule(a, 8.0, 1.0, 1.0, 20.0, 2, 2, 10) == 4.0
    assert impl.rho_schedule(ab, 1.0, 1.0, 0.0, 100.0, 2, 2, 10) == 1.0


def _gtilde_apply(g, zf, alpha, rho):
    """DctCoupledSolver::apply (operators.cpp:420-446) in numpy."""
    m1, m2, m3 = g.m
    n1, V = m1 + 1, g.h[0] * g.h[1] * g.h[2]
    w2, w3 = alpha * V / g.h[1] ** 2, alpha * V / g.h[2] ** 2
    z = zf.reshape(m3, m2, n1)
    o = rho * V * z
    o[:, 1:] += w2 * (z[:, 1:] - z[:, :-1])
    o[:, :-1] += w2 * (z[:, :-1] - z[:, 1:])
    if m3 > 1:
        o[1:] += w3 * (z[1:] - z[:-1])
        o[:-1] += w3 * (z[:-1] - z[1:])
    return o.ravel()


def kat_z_update(impl):
    # test_admm.cpp:260-296
    g = abi.Grid.make(6, 5, 4, h=(0.5, 1.0, 1.5))
    rng = np.random.default_rng(79)
    b, u = rng.uniform(-1, 1, g.faces), rng.uniform(-1, 1, g.faces)
    z0 = impl.z_update(g, b, u, 3.0, 1e-30)
    assert np.allclose(z0, b + u, rtol=1e-9, atol=0)
    zc = impl.z_update(g, np.full(g.faces, 1.5), np.full(g.faces, 0.75), 3.0, 7.0)
    assert np.allclose(zc, 2.25, rtol=1e-12, atol=0)
    z = impl.z_update(g, b, u, 3.0, 7.0)
    w = 3.0 * g.h[0] * g.h[1] * g.h[2]
    rhs = w * (b + u)
    res = _gtilde_apply(g, z, 7.0, 3.0) - rhs
    assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(rhs)


def kat_dct_solve(impl):
    # test_operators.cpp:229-262: zero -> 0, constant -> c/(rho V), residual
    g = abi.Grid.make(7, 6, 5, h=(1.0, 0.8, 1.2))
    V = g.h[0] * g.h[1] * g.h[2]
    out = impl.dct_solve(g, np.zeros(g.faces), 5.0, 2.0)
    out = out[1] if isinstance(out, tuple) else out
    assert not np.any(out)
    c = impl.dct_solve(g, np.full(g.faces, 3.0), 5.0, 2.0)
    c = c[1] if isinstance(c, tuple) else c
    assert np.allclose(c, 3.0 / (2.0 * V), rtol=1e-12)
    rng = np.random.default_rng(5)
    rhs = rng.uniform(-1, 1, g.faces)
    z = impl.dct_solve(g, rhs, 5.0, 2.0)
    z = z[1] if isinstance(z, tuple) else z
    assert np.linalg.norm(_gtilde_apply(g, z, 5.0, 2.0) - rhs) <= 1e-10 * np.linalg.norm(rhs)


def kat_b_update_identities(impl):
    # test_admm.cpp:155-176: identical images, zero state -> b stays exactly 0
    g = abi.Grid.make(8, 6, 1)
    d = synth.make_pair(synth.SynthSpec(m=(8, 6, 1), seed=1, scale=400.0))
    z = np.zeros(g.faces)
    r = impl.b_update(g, d.iplus, d.iplus.copy(), z, z, z, 100.0)
    assert not np.any(r["b"])
    # test_admm.cpp:178-210: zero images -> one SQP step = tridiagonal solve
    g = abi.Grid.make(6, 4, 1)
    zero = np.zeros(g.cells)
    rng = np.random.default_rng(78)
    zz = rng.uniform(-0.05, 0.05, g.faces)
    params = abi.ObjectiveParams(5.0, 10.0, 1e-3)
    r = impl.b_update(g, zero, zero, np.zeros(g.faces), zz, np.zeros(g.faces), 50.0,
                      params=params, cfg=abi.AdmmConfig(sqp_max_iter=1))
    n1, V = g.n1, 1.0
    T = np.zeros((n1, n1))
    w = 5.0 * V
    for i in range(n1 - 1):
        T[i, i] += w
        T[i + 1, i + 1] += w
        T[i, i + 1] -= w
        T[i + 1, i] -= w
    T += 50.0 * V * np.eye(n1)
    expect = np.concatenate([np.linalg.solve(T, 50.0 * V * zz.reshape(-1, n1)[c])
                             for c in range(g.columns)])
    assert np.allclose(r["b"], expect, rtol=1e-11, atol=1e-14)


def phantom_gaussian(g, amp=400.0):
    """The reference's test phantom (image.cpp:285-305), evaluated in numpy."""
    m1, m2, m3 = g.m
    ext = [m1 * g.h[0], m2 * g.h[1], m3 * g.h[2]]
    c = [0.52 * ext[0], 0.47 * ext[1], 0.5 * ext[2]]
    s = [0.23 * ext[0], 0.34 * ext[1], 0.29 * max(ext[2], g.h[2])]
    x = [(np.arange(m) + 0.5) * h for m, h in zip(g.m, g.h)]
    e = ((x[0][None, None, :] - c[0]) / s[0]) ** 2 + ((x[1][None, :, None] - c[1]) / s[1]) ** 2
    if g.dim == 3:
        e = e + ((x[2][:, None, None] - c[2]) / s[2]) ** 2
    return np.ascontiguousarray((amp * np.exp(-0.5 * e)).ravel())


def kat_b_update_saturation(impl):
    # test_admm.cpp:237-258: pulled past the bound, every cell sits on it exactly
    g = abi.Grid.make(6, 4, 1)
    ip = phantom_gaussian(g)
    z = np.zeros(g.faces)
    for j in range(4):
        for i in range(g.n1):
            z[i + g.n1 * j] = 2.0 * i
    r = impl.b_update(g, ip, ip.copy(), np.zeros(g.faces), z, np.zeros(g.faces), 1e6,
                      params=abi.ObjectiveParams(1e-6, 0.0, 1e-3))
    dd = np.diff(r["b"].reshape(-1, g.n1), axis=1)
    assert np.all(dd <= 1.0) and np.all(dd >= 1.0 - 1e-9)
    assert r["kkt_violation"] <= 1e-8


def kat_pcg_zero_gradient(impl):
    g = abi.Grid.make(6, 4, 1)
    z = np.zeros(g.faces)
    d = np.zeros(g.cells)
    r = impl.pcg(g, d, d, z, z, 0.1, 10)
    assert r["iters"] == 0 and r["reached_tol"] and not np.any(r["d"])


def kat_block_precond_exact(impl):
    # test_gn_pcg.cpp:141-160: with a column-separable Hessian (2D, m2 = 1 not
    # allowed -> alpha tiny cross weights) the block preconditioner solves the
    # system in one PCG iteration when cross coupling vanishes: use a grid
    # whose perpendicular spacing makes w2 negligible.
    g = abi.Grid.make(8, 2, 1, h=(1.0, 1e8, 1.0))
    d = synth.make_pair(synth.SynthSpec(m=(8, 2, 1), seed=3, scale=400.0))
    b = np.zeros(g.faces)
    grad = impl.objective_gn(g, d.iplus, d.iminus, b)["grad"]
    r = impl.pcg(g, d.iplus, d.iminus, b, grad, 1e-6, 10)
    assert r["iters"] == 1


def kat_objective_values(impl):
    # objective_gn parts: identical images at b = 0 -> everything zero
    g = abi.Grid.make(8, 6, 4)
    d = synth.make_pair(synth.SynthSpec(m=(8, 6, 4), seed=3, scale=400.0))
    r = impl.objective_gn(g, d.iplus, d.iplus.copy(), np.zeros(g.faces))
    assert r["feasible"] and r["value"] == 0.0 and r["dist"] == 0.0 and not np.any(r["grad"])
    # penalty pole: |D1 b| = 1 exactly -> infeasible
    b = np.zeros(g.faces)
    b.reshape(-1, g.n1)[:, 1:] = 1.0
    assert not impl.objective_gn(g, d.iplus, d.iminus, b)["feasible"]


ALL = [kat_qp_two_face, kat_qp_cycling_guard, kat_qp_brute_force, kat_dual_update,
       kat_rho_schedule, kat_z_update, kat_dct_solve, kat_b_update_identities,
       kat_b_update_saturation, kat_pcg_zero_gradient, kat_block_precond_exact,
       kat_objective_values]
