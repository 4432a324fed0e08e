"""ADMM hot path on the GPU vs the oracle (the C restatement of the
reference, bitwise pinned to it): b-step, z-step, dual update, the full
admm_solve loop, and batched column QPs. All through the C ABI."""
import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth

pytestmark = pytest.mark.gpu

EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


def small_pair(m=(16, 12, 8), seed=7, scale=1.0):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=seed))
    return d.grid, d.iplus * scale, d.iminus * scale


def state_after(oracle, g, ip, im, iters, scale_cfg=None):
    cfg = abi.AdmmConfig(max_iter=iters, **EXACT)
    r = oracle.admm_solve(g, ip, im, cfg=cfg)
    return r


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_b_update_bitwise(ctx, oracle, scale):
    g, ip, im = small_pair(scale=scale)
    st = state_after(oracle, g, ip, im, 6)
    for rho in (st["rho"], 1e6, 100.0):
        ref = oracle.b_update(g, ip, im, st["b"], st["z"], st["u"], rho)
        out = ctx.b_update(g, ip, im, st["b"], st["z"], st["u"], rho)
        assert ref["rc"] == 0
        assert np.array_equal(out["b"], ref["b"]), np.abs(out["b"] - ref["b"]).max()
        assert out["sqp_iters"] == ref["sqp_iters"]
        assert out["qp_iters"] == ref["qp_iters"]
        assert out["kkt_violation"] == ref["kkt_violation"]


def test_z_update_bitwise(ctx, oracle):
    g, ip, im = small_pair()
    rng = np.random.default_rng(3)
    b, u = rng.uniform(-1, 1, g.faces), rng.uniform(-1, 1, g.faces)
    for rho, alpha in ((3.0, 7.0), (1e6, 50.0), (100.0, 50.0)):
        ref = oracle.z_update(g, b, u, rho, alpha)
        out = ctx.z_update(g, b, u, rho, alpha)
        assert np.array_equal(out, ref), np.abs(out - ref).max()


def test_z_update_2d_and_anisotropic(ctx, oracle):
    rng = np.random.default_rng(4)
    for g in (abi.Grid.make(6, 5, 4, h=(0.5, 1.0, 1.5)), abi.Grid.make(12, 10, 1),
              abi.Grid.make(7, 33, 19, h=(1.0, 0.7, 1.3))):
        b, u = rng.uniform(-1, 1, g.faces), rng.uniform(-1, 1, g.faces)
        ref = oracle.z_update(g, b, u, 3.0, 7.0)
        out = ctx.z_update(g, b, u, 3.0, 7.0)
        assert np.array_equal(out, ref), (g.dims(), np.abs(out - ref).max())


def test_dual_update(ctx, oracle):
    g, _, _ = small_pair()
    rng = np.random.default_rng(5)
    b, zn, zo, uo = (rng.uniform(-1, 1, g.faces) for _ in range(4))
    u_ref, r_ref = oracle.dual_update(g, b, zn, zo, uo, 2.0, 0.2, 0.2)
    u_out, r_out = ctx.dual_update(g, b, zn, zo, uo, 2.0, 0.2, 0.2)
    assert np.array_equal(u_out, u_ref)
    for k in r_ref:
        assert r_out[k] == pytest.approx(r_ref[k], rel=1e-13)


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_admm_solve_small_bitwise(ctx, oracle, scale):
    g, ip, im = small_pair(scale=scale)
    cfg = abi.AdmmConfig(max_iter=20, **EXACT)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    out = ctx.admm_solve(g, ip, im, cfg=cfg)
    assert out["stop"] == ref["stop"] and len(out["rows"]) == len(ref["rows"])
    assert np.array_equal(out["b"], ref["b"]), np.abs(out["b"] - ref["b"]).max()
    assert np.array_equal(out["z"], ref["z"])
    assert np.array_equal(out["u"], ref["u"])
    assert out["rho"] == ref["rho"]
    for a, r in zip(out["rows"], ref["rows"]):
        assert a["rho"] == r["rho"]
        assert a["kkt_violation"] == r["kkt_violation"]
        for k in ("primal_res", "dual_res", "eps_pri", "eps_dual", "lagrangian"):
            assert a[k] == pytest.approx(r[k], rel=1e-12, abs=1e-300), k


@pytest.mark.parametrize("m,h,scale", [((512, 6, 4), (1.0, 1.0, 1.0), 1.0),
                                       ((512, 6, 4), (1.0, 1.0, 1.0), 400.0),
                                       ((301, 5, 3), (0.7, 1.3, 0.9), 1.0)])
def test_admm_solve_long_columns_bitwise(ctx, oracle, m, h, scale):
    """Long phase-encoding columns (n1 = 513 as in C5, and an odd n1 with a
    non-power-of-two h1, i.e. the exact-division path): the b-step's shared-
    memory layout, its chain helpers and every certified shortcut against the
    oracle, bitwise."""
    d = synth.make_pair(synth.SynthSpec(m=m, seed=13))
    g = abi.Grid.make(*m, h=h)  # the spacing only rescales the same arrays
    ip, im = d.iplus * scale, d.iminus * scale
    cfg = abi.AdmmConfig(max_iter=8, **EXACT)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    out = ctx.admm_solve(g, ip, im, cfg=cfg)
    assert out["stop"] == ref["stop"] and len(out["rows"]) == len(ref["rows"])
    for k in ("b", "z", "u"):
        assert np.array_equal(out[k], ref[k]), k
    for a, r in zip(out["rows"], ref["rows"]):
        assert a["rho"] == r["rho"] and a["kkt_violation"] == r["kkt_violation"]


def test_admm_solve_default_tolerances_stop_early(ctx, oracle):
    g, ip, im = small_pair()
    ref = oracle.admm_solve(g, ip, im)
    out = ctx.admm_solve(g, ip, im)
    assert out["stop"] == ref["stop"]
    assert len(out["rows"]) == len(ref["rows"])
    assert np.array_equal(out["b"], ref["b"])


def test_qp_batch_matches_oracle(ctx, oracle):
    rng = np.random.default_rng(77)
    n, h, nqp = 5, 0.8, 200
    gd = 2.5 + rng.uniform(-1, 1, (nqp, n))
    go = np.zeros((nqp, n))
    go[:, :-1] = 0.9 * rng.uniform(-1, 1, (nqp, n - 1))
    c = 4.0 * rng.uniform(-1, 1, (nqp, n))
    x0 = np.zeros((nqp, n))
    out = ctx.qp_active_set_batch(n, h, gd, go, c, x0, 200)
    for q in range(nqp):
        ref = oracle.qp_active_set(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), x0[q].copy(), 200)
        assert out["status"][q] == ref["rc"] == 0
        assert np.array_equal(out["x"][q], ref["x"])
        assert np.array_equal(out["lam"][q], ref["lam"])
        assert np.array_equal(out["sign"][q], ref["sign"])
        assert out["iters"][q] == ref["iters"]
        kk = oracle.verify_qp_kkt(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), ref["x"], ref["lam"], ref["sign"])
        assert out["kkt"][q] == kk


def test_qp_goldens(ctx):
    # test_admm.cpp:101-124: unconstrained optimum [3,-3] clamps to [0.5,-0.5], lambda 2.5
    out = ctx.qp_active_set_batch(2, 1.0, [1, 1], [0, 0], [-3, 3], [0, 0], 50)
    assert out["x"][0] == pytest.approx([0.5, -0.5], rel=1e-12)
    assert out["sign"][0][0] == 1
    assert out["lam"][0][0] == pytest.approx(2.5, rel=1e-12)
    assert out["kkt"][0] <= 1e-10
    # infeasible start is rejected (std::invalid_argument)
    out = ctx.qp_active_set_batch(2, 1.0, [1, 1], [0, 0], [0, 0], [0, 5.0], 50)
    assert out["status"][0] == abi.EPC_ERR_INVALID_ARGUMENT
    # cycling guard trips at the cap (test_admm.cpp:149-153)
    out = ctx.qp_active_set_batch(3, 1.0, [1, 1, 1], [0, 0, 0], [-9, 0, 9], [0, 0, 0], 1)
    assert out["status"][0] == abi.EPC_ERR_RUNTIME
    assert "cycling guard" in out["message"]


@pytest.mark.slow
def test_admm_c1_bitwise(ctx, oracle):
    d = synth.make_config("C1")
    cfg = abi.AdmmConfig(max_iter=50, **EXACT)
    ref = oracle.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    out = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    rel = np.linalg.norm(out["b"] - ref["b"]) / np.linalg.norm(ref["b"])
    assert rel <= 1e-8
    assert np.array_equal(out["b"], ref["b"])
    for a, r in zip(out["rows"], ref["rows"]):
        assert a["lagrangian"] == pytest.approx(r["lagrangian"], rel=1e-9)


@pytest.mark.slow
def test_admm_c3_bench_config_bitwise_vs_reference(ctx):
    """The bench's own workload (BASELINE configs[2], 256x256x96) against the
    compiled reference library itself (oracle/_ref, all host threads) for the
    first 3 ADMM iterations: b, z, u, rho and every row bitwise."""
    import os
    from oracle import ffi
    if not ffi.available("ref"):
        pytest.skip("reference library not available")
    ref = ffi.load("ref")
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    d = synth.make_config("C3")
    cfg = abi.AdmmConfig(max_iter=3, threads=threads, **EXACT)
    r = ref.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    o = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    for k in ("b", "z", "u"):
        assert np.array_equal(o[k], r[k]), k
    assert o["rho"] == r["rho"] and o["stop"] == r["stop"]
    for a, b in zip(o["rows"], r["rows"]):
        assert a["rho"] == b["rho"] and a["kkt_violation"] == b["kkt_violation"]
        assert a["lagrangian"] == pytest.approx(b["lagrangian"], rel=1e-12)


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_bstep_modes_bitwise(ctx, oracle, scale):
    """The certified-enclosure b-step (default), the diagnostic instantiation
    with counters, and the all-chains mode all return the reference's b, and
    their line searches make the same decisions (same trial counts)."""
    from paper_1607_00531_b200.epicorr import Context
    g, ip, im = small_pair(scale=scale)
    st = state_after(oracle, g, ip, im, 4)
    ref = oracle.b_update(g, ip, im, st["b"], st["z"], st["u"], st["rho"])
    counters = {}
    try:
        for name, bits in (("prod", 0), ("diag", Context.MODE_BSTEP_TIMING),
                           ("chained", Context.MODE_BSTEP_TIMING | Context.MODE_BSTEP_CHAINED)):
            ctx.set_mode(0)  # counters reset when timing is switched on
            ctx.set_mode(bits)
            out = ctx.b_update(g, ip, im, st["b"], st["z"], st["u"], st["rho"])
            assert np.array_equal(out["b"], ref["b"]), (name, np.abs(out["b"] - ref["b"]).max())
            assert out["sqp_iters"] == ref["sqp_iters"] and out["qp_iters"] == ref["qp_iters"]
            if bits:
                counters[name] = ctx.bstep_counters()
    finally:
        ctx.set_mode(0)
    d, c = counters["diag"], counters["chained"]
    assert d["ls_trials"] == c["ls_trials"] and d["ls_searches"] == c["ls_searches"]
    assert c["ls_undecided"] == 0 and 0 <= d["ls_undecided"] <= d["ls_trials"]
    hist = sum(d[k] for k in ("acc0", "acc1", "acc2_3", "acc4_7", "acc8_15", "acc16_31",
                              "acc32_39", "fail"))
    assert hist == d["ls_searches"]


@pytest.mark.parametrize("alpha,rho", [(1e4, 1e-2), (50.0, 100.0), (1e-3, 1e6), (2e5, 1.0)])
def test_b_update_segmented_chains_bitwise(ctx, oracle, alpha, rho):
    """The LDL^T chain and the sweeps run as 32-lane segments with agreement
    rounds (csrc/bstep.cu, seg_factor / seg_sweep). A large alpha / rho ratio
    makes G nearly a Laplacian, whose recurrences barely contract, so the
    segments need many rounds or fall back to the one-thread chains; a small
    one makes them agree at once. Every case must match the oracle bitwise,
    at n1 = 257 (9-step segments), n1 = 301 (too long for the 9-step segments of the staged-image kernel:
    one-thread chains) and n1 = 513 (long-column kernel, 17-step segments)."""
    for m in ((256, 4, 3), (300, 3, 2), (512, 3, 2)):
        g, ip, im = small_pair(m=m, seed=11)
        st = state_after(oracle, g, ip, im, 3)
        params = abi.ObjectiveParams(alpha=alpha)
        ref = oracle.b_update(g, ip, im, st["b"], st["z"], st["u"], rho, params=params)
        assert ref["rc"] == 0, ref
        out = ctx.b_update(g, ip, im, st["b"], st["z"], st["u"], rho, params=params)
        assert np.array_equal(out["b"], ref["b"]), (m, np.abs(out["b"] - ref["b"]).max())
        assert out["sqp_iters"] == ref["sqp_iters"] and out["qp_iters"] == ref["qp_iters"]
        assert out["kkt_violation"] == ref["kkt_violation"]


@pytest.mark.parametrize("n,amp", [(60, 40.0), (200, 60.0), (257, 200.0)])
def test_qp_large_active_sets_bitwise(ctx, oracle, n, amp):
    """QPs whose active sets grow to tens of rows (as the x400 columns' do),
    so the Schur systems are solved by the whole warp (warp_spd_solve: the
    right-looking Cholesky whose every entry keeps the reference's ascending-k
    chain) and p = w + sum_r lambda_r q_r runs four chains per lane: x,
    lambda, signs, iteration counts and the KKT value bitwise vs the oracle."""
    rng = np.random.default_rng(n)
    nqp, h = 12, 1.0
    gd = 3.0 + rng.uniform(0, 1, (nqp, n))
    go = np.zeros((nqp, n))
    go[:, :-1] = -1.0 + 0.2 * rng.uniform(-1, 1, (nqp, n - 1))
    c = amp * np.cumsum(rng.uniform(-1, 1, (nqp, n)), axis=1) / np.sqrt(n)
    x0 = np.zeros((nqp, n))
    out = ctx.qp_active_set_batch(n, h, gd, go, c, x0, 6 * n + 10)
    most = 0
    for q in range(nqp):
        ref = oracle.qp_active_set(n, h, gd[q].copy(), go[q].copy(), c[q].copy(), x0[q].copy(),
                                   6 * n + 10)
        assert out["status"][q] == ref["rc"], q
        if ref["rc"] != 0:
            continue
        assert np.array_equal(out["x"][q], ref["x"]), q
        assert np.array_equal(out["lam"][q], ref["lam"]), q
        assert np.array_equal(out["sign"][q], ref["sign"]), q
        assert out["iters"][q] == ref["iters"], q
        most = max(most, int(np.count_nonzero(ref["sign"])))
    assert most >= 10, most  # the Schur path really ran with sizable systems
