"""The pipelined ADMM loop (EPC_MODE_DEVICE_LOOP: stop / rho decisions on
the device, one iteration in flight, api.cu k_admm_decide) against the
synchronous default loop (every iteration read back, decisions on the host):
identical fields, rho, stops, messages and rows (the timing fields aside),
for single pairs that stop early or run to the cap, and for a batch whose
pairs stop at different iterations or fail."""
import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth
from paper_1607_00531_b200.epicorr import Context

pytestmark = pytest.mark.gpu

ROW_KEYS = ("level", "iter", "rho", "kkt_violation", "primal_res", "dual_res", "eps_pri",
            "eps_dual", "lagrangian")


def both(ctx, fn):
    """(device loop, synchronous loop) results of fn"""
    ctx.set_mode(Context.MODE_DEVICE_LOOP)
    try:
        out = fn()
    finally:
        ctx.set_mode(0)
    return out, fn()


def same_rows(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        for k in ROW_KEYS:
            assert x[k] == y[k], k


@pytest.mark.parametrize("scale,tol", [(1.0, None), (400.0, None), (1.0, 1e-300), (3.0, 0.05)])
def test_pipelined_loop_matches_sync_loop(ctx, scale, tol):
    d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=7))
    g, ip, im = d.grid, d.iplus * scale, d.iminus * scale
    cfg = abi.AdmmConfig(max_iter=30) if tol is None else abi.AdmmConfig(max_iter=30, eps_abs=tol,
                                                                          eps_rel=tol)
    out, ref = both(ctx, lambda: ctx.admm_solve(g, ip, im, cfg=cfg))
    assert out["stop"] == ref["stop"] and out["message"] == ref["message"]
    assert out["rho"] == ref["rho"]
    for k in ("b", "z", "u"):
        assert np.array_equal(out[k], ref[k]), k
    same_rows(out["rows"], ref["rows"])


def test_pipelined_batch_matches_sync_loop(ctx):
    m = (16, 12, 8)
    g, ip, im = synth.make_batch("C4", npairs=3, m=m)
    nc = g.cells
    ips = [ip[q * nc:(q + 1) * nc].copy() for q in range(3)]
    ims = [im[q * nc:(q + 1) * nc].copy() for q in range(3)]
    bad = ips[0].copy()
    bad[16 * 5 + 3] = np.nan  # column 5 fails at iteration 1
    ips += [ips[0] * 400.0, bad, ips[1] * 20.0]
    ims += [ims[0] * 400.0, ims[0].copy(), ims[1] * 20.0]
    P = len(ips)
    cfg = abi.AdmmConfig(max_iter=40)
    cip, cim = np.concatenate(ips), np.concatenate(ims)
    out, ref = both(ctx, lambda: ctx.admm_solve_batch(g, P, cip, cim, cfg=cfg))
    for k in ("b", "z", "u"):
        assert np.array_equal(out[k], ref[k]), k
    for o, r in zip(out["pairs"], ref["pairs"]):
        assert o["stop"] == r["stop"] and o["message"] == r["message"] and o["rho"] == r["rho"]
        same_rows(o["rows"], r["rows"])
    assert out["pairs"][4]["stop"] == abi.STOP_ERROR


def test_pipelined_counters_match(ctx):
    """The decision counters (certified / exact) and the SQP / QP totals are
    the same either way, also with every decision on the sequential sums."""
    d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=3))
    cfg = abi.AdmmConfig(max_iter=20, eps_abs=1e-300, eps_rel=1e-300)
    for extra in (0, Context.MODE_EXACT_SUMS):
        counts = []
        for mode in (extra, extra | Context.MODE_DEVICE_LOOP):
            ctx.set_mode(mode)
            try:
                c0 = ctx.admm_counters()
                ctx.admm_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
                c1 = ctx.admm_counters()
            finally:
                ctx.set_mode(0)
            counts.append([b - a for a, b in zip(c0, c1)])
        assert counts[0] == counts[1], (extra, counts)
        assert sum(counts[0][:2]) == 20
