"""Multilevel (proj/src/multilevel.cpp) on CPU:
  * the reference's own expectations (tests/test_multilevel.cpp, restated)
    on the oracle, on the reference library when present, and on the
    product's host-only default_schedule;
  * the oracle restatement bitwise against the live reference library for
    restrict_image, prolong_field and multilevel_solve (GN and the three ADMM
    restarts), where the reference tree is present.
The GPU side is tests/test_gpu_multilevel.py."""
import numpy as np
import pytest

from kats import phantom_gaussian
from oracle import ffi
from paper_1607_00531_b200 import abi, epicorr, synth

EXACT = dict(eps_abs=1e-300, eps_rel=1e-300)
needs_ref = pytest.mark.skipif(not ffi.available("ref"), reason="reference library not available")


def g2(m1, m2, h1=1.0, h2=1.0):
    return abi.Grid.make(m1, m2, 1, h=(h1, h2, 1.0))


def impls():
    out = [("oracle", ffi.load("oracle"))]
    if ffi.available("ref"):
        out.append(("ref", ffi.load("ref")))
    return out


@pytest.mark.parametrize("kind", ["oracle", "ref", "product"])
def test_default_schedule_expectations(kind):
    if kind == "ref" and not ffi.available("ref"):
        pytest.skip("reference library not available")
    sched = epicorr.default_schedule if kind == "product" else ffi.load(kind).default_schedule
    s = sched(g2(128, 128))
    assert [g.m[0] for g in s] == [16, 32, 64, 128]
    assert all(g.m[0] * g.h[0] == pytest.approx(128.0) for g in s)
    s = sched(abi.Grid.make(96, 96, 64))
    assert [list(g.m) for g in s[:2]] == [[24, 24, 16], [48, 48, 32]] and len(s) == 3
    s = sched(abi.Grid.make(50, 50, 33, h=(1.0, 1.0, 2.0)))
    assert list(s[0].m) == [25, 25, 17] and s[0].m[2] * s[0].h[2] == pytest.approx(66.0)


@pytest.mark.parametrize("name,impl", impls())
def test_restrict_expectations(name, impl):
    f, c = g2(8, 6), g2(4, 3, 2.0, 2.0)
    r = impl.restrict_image(f, c, np.full(f.cells, 3.5))
    assert np.allclose(r, 3.5, rtol=1e-14, atol=0)
    f4, c2 = g2(4, 4, 0.25, 0.25), g2(2, 2, 0.5, 0.5)
    img = np.empty(16)
    for j in range(4):
        for i in range(4):
            img[i + 4 * j] = (1 if j < 2 else 5) if i < 2 else (3 if j < 2 else 7)
    assert np.allclose(impl.restrict_image(f4, c2, img), [1.0, 3.0, 5.0, 7.0])
    same = impl.restrict_image(c2, c2, np.array([1.0, 3.0, 5.0, 7.0]))
    assert np.array_equal(same, [1.0, 3.0, 5.0, 7.0])       # same grid: identity
    for f, c in ((g2(32, 16, 0.5, 1.0), g2(16, 8, 1.0, 2.0)),
                 (g2(33, 17), g2(17, 9, 33.0 / 17.0, 17.0 / 9.0))):  # exact and partial tiling
        img = phantom_gaussian(f)
        r = impl.restrict_image(f, c, img)
        vf = f.h[0] * f.h[1] * f.h[2]
        vc = c.h[0] * c.h[1] * c.h[2]
        assert np.sum(r * vc) == pytest.approx(np.sum(img * vf), rel=1e-12)
    with pytest.raises(ValueError):
        impl.restrict_image(g2(8, 8), g2(16, 16, 0.5, 0.5), np.zeros(64))


@pytest.mark.parametrize("name,impl", impls())
def test_prolong_expectations(name, impl):
    c, f = g2(8, 8, 2.0, 2.0), g2(16, 16)
    assert np.allclose(impl.prolong_field(c, f, np.full(c.faces, 1.75)), 1.75, rtol=1e-14, atol=0)
    lin = np.empty(c.faces)
    for j in range(8):
        for i in range(9):
            lin[i + 9 * j] = 0.25 * (i * 2.0) + 2.0
    pl = impl.prolong_field(c, f, lin)
    want = np.array([0.25 * i + 2.0 for j in range(16) for i in range(17)])
    assert np.allclose(pl, want, rtol=1e-13, atol=0)
    steep = np.empty(c.faces)
    for j in range(8):
        for i in range(9):
            steep[i + 9 * j] = (1.1 if j == 3 else 0.999) * (i * 2.0)
    resc = impl.prolong_field(c, f, steep).reshape(16, 17)
    assert np.abs(np.diff(resc, axis=1)).max() == pytest.approx(0.95, rel=1e-12)
    with pytest.raises(ValueError):
        impl.prolong_field(f, c, np.zeros(f.faces))


def _rand_field(g, seed, scale=0.3):
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, g.faces).cumsum() * 0.0 + rng.uniform(-scale, scale, g.faces)


RESTRICT_CASES = [(abi.Grid.make(12, 10, 8), abi.Grid.make(6, 5, 4, h=(2.0, 2.0, 2.0))),
                  (abi.Grid.make(13, 11, 7), abi.Grid.make(7, 6, 4, h=(13 / 7, 11 / 6, 7 / 4))),
                  (g2(33, 17), g2(17, 9, 33.0 / 17.0, 17.0 / 9.0))]


@needs_ref
@pytest.mark.parametrize("fine,coarse", RESTRICT_CASES)
def test_oracle_restrict_prolong_bitwise_vs_reference(fine, coarse):
    orc, ref = ffi.load("oracle"), ffi.load("ref")
    img = np.random.default_rng(3).uniform(0.0, 2.0, fine.cells)
    assert np.array_equal(orc.restrict_image(fine, coarse, img), ref.restrict_image(fine, coarse, img))
    b = np.random.default_rng(4).uniform(-0.3, 0.3, coarse.faces)
    assert np.array_equal(orc.prolong_field(coarse, fine, b), ref.prolong_field(coarse, fine, b))
    steep = np.random.default_rng(5).uniform(-3.0, 3.0, coarse.faces)   # rescue path
    assert np.array_equal(orc.prolong_field(coarse, fine, steep),
                          ref.prolong_field(coarse, fine, steep))


def _ml_case():
    d = synth.make_pair(synth.SynthSpec(m=(24, 20, 16), seed=21))
    return d.grid, d.iplus, d.iminus


@needs_ref
@pytest.mark.parametrize("solver,restart", [(abi.SOLVER_GN, abi.RESTART_AVERAGE),
                                            (abi.SOLVER_ADMM, abi.RESTART_PROLONG_ALL),
                                            (abi.SOLVER_ADMM, abi.RESTART_B_FOR_BOTH),
                                            (abi.SOLVER_ADMM, abi.RESTART_AVERAGE)])
def test_oracle_multilevel_bitwise_vs_reference(solver, restart):
    g, ip, im = _ml_case()
    orc, ref = ffi.load("oracle"), ffi.load("ref")
    levels = orc.default_schedule(g, max_levels=3, min_cells=4)
    kw = dict(gn_cfg=abi.GnConfig(max_outer=3), admm_cfg=abi.AdmmConfig(max_iter=6, **EXACT),
              restart=restart, admm_max_iter=[3, 4, None])
    a = orc.multilevel_solve(g, ip, im, levels, solver, **kw)
    b = ref.multilevel_solve(g, ip, im, levels, solver, **kw)
    assert a["stop"] == b["stop"] and a["b_level"] == b["b_level"]
    assert np.array_equal(a["b"], b["b"])
    rows = "gn_rows" if solver == abi.SOLVER_GN else "admm_rows"
    assert len(a[rows]) == len(b[rows])
    for x, y in zip(a[rows], b[rows]):
        assert x["level"] == y["level"] and x["iter"] == y["iter"]
        key = "j_value" if solver == abi.SOLVER_GN else "rho"
        assert x[key] == y[key]
