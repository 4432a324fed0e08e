"""Multilevel on the GPU (epc_restrict_image / epc_prolong_field /
epc_multilevel_solve) against the oracle, which test_multilevel.py pins
bitwise to the reference: restriction and prolongation bitwise; ADMM
multilevel bitwise in b for every restart; GN multilevel within the
north-star tolerance (the GN solve is not bitwise, ~1e-14)."""
import numpy as np
import pytest
import torch

from paper_1607_00531_b200 import abi, synth
from test_multilevel import RESTRICT_CASES, EXACT, g2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fine,coarse", RESTRICT_CASES + [(g2(8, 6), g2(4, 3, 2.0, 2.0))])
def test_restrict_prolong_bitwise(ctx, oracle, fine, coarse):
    img = np.random.default_rng(3).uniform(0.0, 2.0, fine.cells)
    assert np.array_equal(ctx.restrict_image(fine, coarse, img),
                          oracle.restrict_image(fine, coarse, img))
    for seed, sc in ((4, 0.3), (5, 3.0)):  # plain and rescued
        b = np.random.default_rng(seed).uniform(-sc, sc, coarse.faces)
        assert np.array_equal(ctx.prolong_field(coarse, fine, b),
                              oracle.prolong_field(coarse, fine, b))
    # device memory path
    dev = torch.device("cuda", 0)
    out = ctx.restrict_image(fine, coarse, torch.from_numpy(img).to(dev)).cpu().numpy()
    assert np.array_equal(out, oracle.restrict_image(fine, coarse, img))


@pytest.mark.parametrize("solver,restart", [(abi.SOLVER_ADMM, abi.RESTART_PROLONG_ALL),
                                            (abi.SOLVER_ADMM, abi.RESTART_B_FOR_BOTH),
                                            (abi.SOLVER_ADMM, abi.RESTART_AVERAGE),
                                            (abi.SOLVER_GN, abi.RESTART_AVERAGE)])
def test_multilevel_matches_reference(ctx, oracle, solver, restart):
    d = synth.make_pair(synth.SynthSpec(m=(32, 24, 16), seed=21))
    g, ip, im = d.grid, d.iplus, d.iminus
    levels = oracle.default_schedule(g, max_levels=3, min_cells=4)
    kw = dict(gn_cfg=abi.GnConfig(max_outer=3), admm_cfg=abi.AdmmConfig(max_iter=8, **EXACT),
              restart=restart, admm_max_iter=[4, 5, None])
    got = ctx.multilevel_solve(g, ip, im, levels, solver, **kw)
    ref = oracle.multilevel_solve(g, ip, im, levels, solver, **kw)
    assert got["stop"] == ref["stop"] and got["b_level"] == ref["b_level"]
    if solver == abi.SOLVER_ADMM:
        assert np.array_equal(got["b"], ref["b"])
        assert [(r["level"], r["iter"], r["rho"]) for r in got["admm_rows"]] == \
               [(r["level"], r["iter"], r["rho"]) for r in ref["admm_rows"]]
    else:
        rel = np.linalg.norm(got["b"] - ref["b"]) / np.linalg.norm(ref["b"])
        assert rel <= 1e-8, rel
        for x, y in zip(got["gn_rows"], ref["gn_rows"]):
            assert x["level"] == y["level"] and x["iter"] == y["iter"]
            assert x["j_value"] == pytest.approx(y["j_value"], rel=1e-9)
