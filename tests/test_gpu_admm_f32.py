"""fp32 variant of the ADMM solve (epc_admm_solve_f32; BASELINE configs[2]
"fp64 and an fp32 variant", SURVEY 8(d) "fp32: reported separately against
the fp64 oracle with a stated tolerance"). Not bitwise: fp32 storage and
element arithmetic, fp64-accumulated sums, QP/SQP thresholds rescaled for
fp32 (admm_f32.cu). Stated tolerances, measured on the synthetic configs:
  * intensity scale 1: b, z within 4e-3 relative L2 of the fp64 oracle at
    30 iterations (24x20x16: 2.9e-3, set by the fp32 arithmetic itself: fp64
    moves only 1.7e-8 there when its inputs are rounded to fp32); at the
    bench's C3 workload (100 iterations) within 3x the fp64 input-rounding
    sensitivity and 5e-3 (measured 4.0e-3 against 1.6e-3); every row's
    Lagrangian within 5e-4 relative (measured 1.4e-4 at 24x20x16, where its
    rho V u.(b - z) terms cancel), the same rho sequence and stop reason. Accumulating the
    fp32 DCT products in fp64 moves the C3 deviation only from 4.0e-3 to
    3.9e-3: the fp32 b-step sets it;
  * intensity x400 (chaotic nonconvex columns): within 4x fp64's own
    input-rounding deviation, final Lagrangian within 5%.
The host- and device-memory paths run the same kernels and agree bitwise."""
import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth

pytestmark = pytest.mark.gpu

EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)


def _case(m, seed, scale=1.0):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=seed, scale=scale))
    return d.grid, d.iplus, d.iminus


def _rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("m", [(24, 20, 16), (40, 30, 1)])
def test_f32_against_fp64_oracle(ctx, oracle, m):
    g, ip, im = _case(m, 5)
    cfg = abi.AdmmConfig(max_iter=30, **EXACT)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    got = ctx.admm_solve_f32(g, ip.astype(np.float32), im.astype(np.float32), cfg=cfg)
    assert got["stop"] == ref["stop"]
    assert _rel(got["b"], ref["b"]) <= 4e-3
    assert _rel(got["z"], ref["z"]) <= 4e-3
    assert len(got["rows"]) == len(ref["rows"])
    for a, b in zip(got["rows"], ref["rows"]):
        assert a["iter"] == b["iter"] and a["rho"] == b["rho"]
        assert a["lagrangian"] == pytest.approx(b["lagrangian"], rel=5e-4)
        assert a["kkt_violation"] <= 1e-4


def test_f32_x400_within_fp64_input_sensitivity(ctx, oracle):
    """At intensity x400 the nonconvex columns are chaotic: fp64 itself moves
    by a few percent when only its inputs are rounded to fp32 (columns settle
    in other local minima). The fp32 solve is held to that scale: b within
    4x the fp64 input-rounding deviation (+1e-3), the final Lagrangian within
    5%, and the same rho sequence over the first 10 iterations."""
    g, ip, im = _case((32, 24, 12), 5, 400.0)
    cfg = abi.AdmmConfig(max_iter=30, **EXACT)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    ip32, im32 = ip.astype(np.float32), im.astype(np.float32)
    refq = oracle.admm_solve(g, ip32.astype(np.float64), im32.astype(np.float64), cfg=cfg)
    got = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
    sens = _rel(refq["b"], ref["b"])
    assert _rel(got["b"], ref["b"]) <= 4 * sens + 1e-3
    assert got["rows"][-1]["lagrangian"] == pytest.approx(ref["rows"][-1]["lagrangian"], rel=5e-2)
    assert [r["rho"] for r in got["rows"][:10]] == [r["rho"] for r in ref["rows"][:10]]


def test_f32_host_and_device_paths_bitwise(ctx):
    torch = pytest.importorskip("torch")
    g, ip, im = _case((20, 16, 10), 7)
    cfg = abi.AdmmConfig(max_iter=8, **EXACT)
    ip32, im32 = ip.astype(np.float32), im.astype(np.float32)
    h = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
    d = ctx.admm_solve_f32(g, torch.from_numpy(ip32).cuda(), torch.from_numpy(im32).cuda(), cfg=cfg)
    for k in ("b", "z", "u"):
        assert np.array_equal(h[k], d[k].cpu().numpy()), k
    assert [r["lagrangian"] for r in h["rows"]] == [r["lagrangian"] for r in d["rows"]]


def test_f32_converges_and_restarts(ctx, oracle):
    """Default tolerances (a converging solve), then a warm restart from the
    returned state with the returned rho (as the multilevel driver does),
    checked against the fp64 oracle restarted from the same state."""
    g, ip, im = _case((16, 12, 8), 3)
    ip32, im32 = ip.astype(np.float32), im.astype(np.float32)
    cfg = abi.AdmmConfig(max_iter=300)
    ref = oracle.admm_solve(g, ip, im, cfg=cfg)
    got = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
    assert got["stop"] == ref["stop"] == 0
    assert abs(len(got["rows"]) - len(ref["rows"])) <= max(2, len(ref["rows"]) // 10)
    cfg2 = abi.AdmmConfig(max_iter=5, **EXACT)
    again = ctx.admm_solve_f32(g, ip32, im32, b=got["b"], z=got["z"], u=got["u"], rho=got["rho"],
                               cfg=cfg2)
    ref2 = oracle.admm_solve(g, ip, im, b=got["b"].astype(np.float64), z=got["z"].astype(np.float64),
                             u=got["u"].astype(np.float64), rho=got["rho"], cfg=cfg2)
    assert again["rows"][0]["rho"] == got["rho"] == ref2["rows"][0]["rho"]
    assert _rel(again["b"], ref2["b"]) <= 2e-3


def test_f32_infeasible_start_raises(ctx):
    g, ip, im = _case((12, 8, 6), 1)
    b = np.zeros(g.faces, np.float32)
    b[1] = 5.0  # |D1 b| > 1
    with pytest.raises(ValueError, match="infeasible"):
        ctx.admm_solve_f32(g, ip.astype(np.float32), im.astype(np.float32), b=b,
                           cfg=abi.AdmmConfig(max_iter=2))


@pytest.mark.slow
def test_f32_c3_bench_config_within_input_rounding_sensitivity(ctx):
    """The stated fp32 tolerance pinned at the bench's own workload (C3,
    256x256x96, 100 iterations). The floor is set by the inputs: the fp64
    solve (bitwise the reference's, tests/test_gpu_fullsize.py) moves by
    `sens` when only I+/I- are rounded to fp32 (measured 1.6e-3), so no
    solver fed fp32 volumes can be held below it. Stated: b and z within
    3 x sens and at most 5e-3 relative L2 of the fp64 result, the same rho
    schedule over the first 30 iterations, final Lagrangian within 1e-4."""
    d = synth.make_config("C3")
    g = d.grid
    cfg = abi.AdmmConfig(max_iter=100, **EXACT)
    ref = ctx.admm_solve(g, d.iplus, d.iminus, cfg=cfg)
    ip32, im32 = d.iplus.astype(np.float32), d.iminus.astype(np.float32)
    refq = ctx.admm_solve(g, ip32.astype(np.float64), im32.astype(np.float64), cfg=cfg)
    got = ctx.admm_solve_f32(g, ip32, im32, cfg=cfg)
    sens = _rel(refq["b"], ref["b"])
    dev_b, dev_z = _rel(got["b"], ref["b"]), _rel(got["z"], ref["z"])
    print(f"C3 fp32: b {dev_b:.3e}, z {dev_z:.3e}, fp64 input-rounding sensitivity {sens:.3e}")
    assert dev_b <= min(3 * sens, 5e-3), (dev_b, sens)
    assert dev_z <= min(3 * sens, 5e-3), (dev_z, sens)
    assert [r["rho"] for r in got["rows"][:30]] == [r["rho"] for r in ref["rows"][:30]]
    assert got["rows"][-1]["lagrangian"] == pytest.approx(ref["rows"][-1]["lagrangian"], rel=1e-4)
