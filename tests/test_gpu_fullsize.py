"""Parity on the BASELINE workloads at their full lengths, against the compiled
reference library itself (oracle/_ref, the unmodified proj/src sources, all
host threads):

  * ADMM C3 (256x256x96, 100 iterations, the bench's workload): b, z, u, rho,
    stop and every row's rho / kkt bitwise over the whole trajectory,
    including the ~25 iterations over which rho walks from 1e6 down to
    rho_min; the rows' residuals within 1e-12 and, with every decision taken
    on the reference's sequential sums (EPC_MODE_EXACT_SUMS), bitwise;
  * ADMM C3 at amplitude x400 (image.hpp:87-90), 20 iterations;
  * GN-PCG C3 (10 GN steps x <= 50 PCG, block-Jacobi, eta 1e-2);
  * the batched solver (C4's entry point): pairs stopping at different
    iterations, at different intensity scales, and one failing column, each
    bitwise against its own single-pair admm_solve;
  * the exact-sums mode at C1.
"""
import os

import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth

pytestmark = pytest.mark.gpu
EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


def _ref():
    from oracle import ffi
    if not ffi.available("ref"):
        pytest.skip("reference library not available")
    ref = ffi.load("ref")
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    return ref, threads


def _check_admm(o, r, rows_exact=False):
    for k in ("b", "z", "u"):
        assert np.array_equal(o[k], r[k]), (k, float(np.abs(o[k] - r[k]).max()))
    assert o["rho"] == r["rho"] and o["stop"] == r["stop"]
    assert len(o["rows"]) == len(r["rows"])
    for a, b in zip(o["rows"], r["rows"]):
        assert a["iter"] == b["iter"] and a["rho"] == b["rho"], a["iter"]
        assert a["kkt_violation"] == b["kkt_violation"], a["iter"]
        assert a["lagrangian"] == pytest.approx(b["lagrangian"], rel=1e-9), a["iter"]
        for f in ("primal_res", "dual_res", "eps_pri", "eps_dual"):
            if rows_exact:
                assert a[f] == b[f], (a["iter"], f)
            else:
                assert a[f] == pytest.approx(b[f], rel=1e-12, abs=1e-300), (a["iter"], f)


@pytest.mark.slow
def test_admm_c3_full_trajectory_bitwise_vs_reference(ctx):
    from paper_1607_00531_b200.epicorr import Context
    ref, threads = _ref()
    d = synth.make_config("C3")
    cfg = abi.AdmmConfig(max_iter=100, threads=threads, **EXACT)
    r = ref.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    rhos = [x["rho"] for x in r["rows"]]
    assert len(set(rhos)) > 5  # the trajectory does walk rho (the window the test is for)
    c0 = ctx.admm_counters()
    o = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    c1 = ctx.admm_counters()
    _check_admm(o, r)
    assert (c1[0] - c0[0]) + (c1[1] - c0[1]) == 100
    try:
        ctx.set_mode(Context.MODE_EXACT_SUMS)
        e = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    finally:
        ctx.set_mode(0)
    _check_admm(e, r, rows_exact=True)
    c2 = ctx.admm_counters()
    assert c2[1] - c1[1] == 100


@pytest.mark.slow
def test_admm_c3_x400_bitwise_vs_reference(ctx):
    ref, threads = _ref()
    d = synth.make_config("C3", scale=400.0)
    cfg = abi.AdmmConfig(max_iter=20, threads=threads, **EXACT)
    r = ref.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    o = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    _check_admm(o, r)
    # the workload is the representative one: the field moves
    assert float(np.abs(r["b"]).max()) > 1.0


@pytest.mark.slow
def test_gn_c3_vs_reference(ctx):
    """gauss_newton_solve (gn_pcg.cpp:197-292) at 256x256x96: b within 1e-8
    relative L2, j_value within 1e-9, equal PCG counts and Wolfe steps."""
    ref, threads = _ref()
    d = synth.make_config("C3")
    cfg = abi.GnConfig(eta=1e-2, max_outer=10, max_pcg=50, eps_obj=1e-300, eps_iter=1e-300,
                       eps_grad=1e-300, precond=abi.PRECOND_BLOCK_JACOBI, threads=threads)
    r = ref.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    o = ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    assert o["stop"] == r["stop"] and len(o["rows"]) == len(r["rows"]) == 11
    rel = np.linalg.norm(o["b"] - r["b"]) / np.linalg.norm(r["b"])
    assert rel <= 1e-8, rel
    for a, b in zip(o["rows"], r["rows"]):
        assert a["pcg_iters"] == b["pcg_iters"], a["iter"]
        assert a["step"] == pytest.approx(b["step"], rel=1e-9), a["iter"]
        assert a["j_value"] == pytest.approx(b["j_value"], rel=1e-9), a["iter"]
    assert sum(x["pcg_iters"] for x in r["rows"]) > 100


@pytest.mark.parametrize("m", [(16, 12, 8), (128, 8, 6)])
def test_admm_batch_pairs_each_bitwise(ctx, oracle, m):
    """epc_admm_solve_batch (C4's entry point) with pairs that stop at
    different iterations under the default tolerances, pairs at different
    intensity scales (x1, x400, x20) and one pair whose column 5 fails
    (a NaN intensity: 'column factor: nonpositive pivot' at iteration 1):
    each pair bitwise against its own admm_solve (admm.cpp:488-560), the
    failed pair's state the one from before the failed iteration.
    At n1 = 129 the forward axis-2 DCT runs in the b-step's drain (layer
    counts over skipped columns of stopped pairs and failing columns)."""
    g, ip, im = synth.make_batch("C4", npairs=3, m=m)
    nc, nf = g.cells, g.faces
    ips = [ip[q * nc:(q + 1) * nc].copy() for q in range(3)]
    ims = [im[q * nc:(q + 1) * nc].copy() for q in range(3)]
    bad = ips[0].copy()
    bad[m[0] * 5 + 3] = np.nan
    ips += [ips[0] * 400.0, bad, ips[1] * 20.0]
    ims += [ims[0] * 400.0, ims[0].copy(), ims[1] * 20.0]
    P = len(ips)
    cfg = abi.AdmmConfig(max_iter=40)
    out = ctx.admm_solve_batch(g, P, np.concatenate(ips), np.concatenate(ims), cfg=cfg)
    stops = set()
    for q in range(P):
        r = oracle.admm_solve(g, ips[q], ims[q], cfg=cfg)
        o = out["pairs"][q]
        assert o["stop"] == r["stop"] and o["message"] == r["message"], q
        assert o["rho"] == r["rho"], q
        for k in ("b", "z", "u"):
            assert np.array_equal(out[k][q * nf:(q + 1) * nf], r[k]), (q, k)
        assert len(o["rows"]) == len(r["rows"]), q
        for a, b in zip(o["rows"], r["rows"]):
            assert a["rho"] == b["rho"] and a["kkt_violation"] == b["kkt_violation"], q
            assert a["lagrangian"] == pytest.approx(b["lagrangian"], rel=1e-12), q
        stops.add((r["stop"], len(r["rows"])))
    assert len(stops) >= 4, stops  # the pairs really end differently
    assert out["pairs"][4]["stop"] == abi.STOP_ERROR
    assert "column 5" in out["pairs"][4]["message"]


def test_admm_batch_warm_start_fixed_count(ctx, oracle):
    """Warm-started batch (per-pair b, z, u, rho) with a fixed iteration
    count: each pair continues exactly as its own warm-started admm_solve."""
    m = (20, 10, 6)
    g, ip, im = synth.make_batch("C4", npairs=3, m=m, scale=3.0)
    nc, nf = g.cells, g.faces
    cfg0 = abi.AdmmConfig(max_iter=4, **EXACT)
    starts = [oracle.admm_solve(g, ip[q * nc:(q + 1) * nc].copy(), im[q * nc:(q + 1) * nc].copy(),
                                cfg=cfg0) for q in range(3)]
    cfg = abi.AdmmConfig(max_iter=12, **EXACT)
    cat = lambda k: np.concatenate([s[k] for s in starts])
    out = ctx.admm_solve_batch(g, 3, ip, im, rho=[s["rho"] for s in starts], cfg=cfg,
                               b=cat("b"), z=cat("z"), u=cat("u"))
    for q in range(3):
        s = starts[q]
        r = oracle.admm_solve(g, ip[q * nc:(q + 1) * nc].copy(), im[q * nc:(q + 1) * nc].copy(),
                              b=s["b"], z=s["z"], u=s["u"], rho=s["rho"], cfg=cfg)
        for k in ("b", "z", "u"):
            assert np.array_equal(out[k][q * nf:(q + 1) * nf], r[k]), (q, k)
        assert out["pairs"][q]["rho"] == r["rho"]


def test_exact_sums_mode_rows_bitwise_c1(ctx, oracle):
    """EPC_MODE_EXACT_SUMS at C1 (50 iterations): every decision on the
    reference's sequential sums (k_seq_sums), the rows' residuals bitwise,
    and the same trajectory as the certified default."""
    from paper_1607_00531_b200.epicorr import Context
    d = synth.make_config("C1")
    cfg = abi.AdmmConfig(max_iter=50, **EXACT)
    r = oracle.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    c0 = ctx.admm_counters()
    try:
        ctx.set_mode(Context.MODE_EXACT_SUMS)
        o = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    finally:
        ctx.set_mode(0)
    c1 = ctx.admm_counters()
    assert c1[1] - c0[1] == 50
    _check_admm(o, r, rows_exact=True)
    o2 = ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    c2 = ctx.admm_counters()
    assert c2[0] - c1[0] == 50  # all certified at C1 (no near-tie)
    _check_admm(o2, r)
