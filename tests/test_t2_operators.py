"""The reference's test-side helpers of the hot path on
CPU: the reference's own expectations (test_operators.cpp:48-214, restated)
on the oracle and, where the reference tree is present, on the reference
library; and the oracle restatement bitwise against the reference for every
helper. The device entry points are in tests/test_gpu_t2_operators.py."""
import numpy as np
import pytest

from oracle import ffi
from paper_1607_00531_b200 import abi, synth

needs_ref = pytest.mark.skipif(not ffi.available("ref"), reason="reference library not available")

GRIDS = [abi.Grid.make(3, 2, 1, h=(0.5, 1.25, 1.0)),
         abi.Grid.make(4, 3, 1, h=(1.0, 0.75, 1.0), origin=(-1.0, 2.0, 0.0)),
         abi.Grid.make(5, 4, 3, h=(0.5, 1.0, 2.0)),
         abi.Grid.make(2, 3, 2)]


def impls():
    out = [("oracle", ffi.load("oracle"))]
    if ffi.available("ref"):
        out.append(("ref", ffi.load("ref")))
    return out


def g2(m1, m2, h1=1.0, h2=1.0):
    return abi.Grid.make(m1, m2, 1, h=(h1, h2, 1.0))


@pytest.mark.parametrize("name,impl", impls())
def test_stencil_examples(name, impl):
    g = g2(2, 2)
    b = np.array([0, 1, 3, 0, 1, 3], dtype=np.float64)
    assert np.allclose(impl.avg_x1(g, b)[:2], [0.5, 2.0], rtol=1e-15, atol=0)
    assert np.all(impl.avg_x1(g, np.full(6, 3.25)) == 3.25)
    b3 = np.array([1, 2, 4, 8, 1, 2, 4, 8], dtype=np.float64)
    assert list(impl.avg_x1(g2(3, 2), b3)[:3]) == [1.5, 3.0, 6.0]
    assert np.allclose(impl.diff_x1(g2(2, 2, 0.5), b)[:2], [2.0, 4.0], rtol=1e-15, atol=0)
    assert np.all(impl.diff_x1(g2(2, 2, 0.5), np.full(6, -7.5)) == 0.0)
    assert list(impl.diff_x1(g2(3, 2), b3)[:3]) == [1.0, 2.0, 4.0]
    out = impl.diff_x1_adjoint(g, np.array([1.0, 1.0, 0.0, 0.0]))
    assert list(out[:3]) == [-1.0, 0.0, 1.0]
    assert not impl.diff_x1_adjoint(g, np.zeros(4)).any()


@pytest.mark.parametrize("name,impl", impls())
@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_adjoint_identity(name, impl, gi):
    g = GRIDS[gi]
    rng = np.random.default_rng(11)
    b, r = rng.uniform(-1, 1, g.faces), rng.uniform(-1, 1, g.cells)
    assert np.dot(impl.diff_x1(g, b), r) == pytest.approx(np.dot(b, impl.diff_x1_adjoint(g, r)),
                                                          rel=1e-12)


@pytest.mark.parametrize("name,impl", impls())
def test_batched_tridiagonal_solve(name, impl):
    g = g2(2, 2)
    rhs = np.random.default_rng(41).uniform(-1, 1, g.faces)
    ident = np.ones(g.faces)
    assert np.array_equal(impl.tridiag_solve_batched(g, ident, np.zeros(g.faces), rhs), rhs)
    d = np.full(g.faces, 2.0)
    off = np.array([-1.0, -1.0, 0.0, -1.0, -1.0, 0.0])
    x = impl.tridiag_solve_batched(g, d, off, np.array([1.0, 0, 0, 1, 0, 0]))
    assert np.allclose(x[:3], [0.75, 0.5, 0.25], rtol=1e-14, atol=0)
    g3 = abi.Grid.make(6, 3, 2)
    rng = np.random.default_rng(42)
    rd = 3.0 + rng.uniform(-1, 1, g3.faces)
    ro = rng.uniform(-1, 1, g3.faces)
    ro.reshape(-1, g3.n1)[:, -1] = 0.0
    r3 = rng.uniform(-1, 1, g3.faces)
    x3 = impl.tridiag_solve_batched(g3, rd, ro, r3)
    res = impl.tridiag_apply(g3, rd, ro, x3, 1.0, np.zeros(g3.faces)) - r3
    assert np.linalg.norm(res) <= 1e-12 * np.linalg.norm(r3)
    bad = np.ones(g.faces)
    bad[1 * g.n1 + 1] = -2.0
    with pytest.raises(RuntimeError, match="column 1"):
        impl.tridiag_solve_batched(g, bad, np.zeros(g.faces), rhs)


@pytest.mark.parametrize("name,impl", impls())
def test_dct_apply_inverts_the_solve(name, impl):
    g = abi.Grid.make(5, 4, 3, h=(0.5, 1.0, 2.0))
    rhs = np.random.default_rng(5).uniform(-1, 1, g.faces)
    rc, z, _ = impl.dct_solve(g, rhs, 3.0, 7.0)
    assert rc == 0
    assert np.linalg.norm(impl.dct_apply(g, z, 3.0, 7.0) - rhs) <= 1e-10 * np.linalg.norm(rhs)


@pytest.mark.parametrize("name,impl", impls())
def test_feasibility(name, impl):
    g = abi.Grid.make(6, 3, 2)
    b = np.zeros(g.faces)
    assert impl.is_strictly_feasible(g, b)
    b.reshape(-1, g.n1)[1, 3] = 1.0 - 1e-11     # |D1 b| just above 1 - kFeasEps
    assert not impl.is_strictly_feasible(g, b)
    b.reshape(-1, g.n1)[1, 3] = 1.0 - 1e-9
    assert impl.is_strictly_feasible(g, b)


def _inputs(g, seed):
    rng = np.random.default_rng(seed)
    d = synth.make_pair(synth.SynthSpec(m=tuple(g.m), seed=seed))
    b = 0.2 * np.cumsum(rng.uniform(-0.1, 0.1, g.faces).reshape(-1, g.n1), axis=1).ravel()
    return dict(b=b, r=rng.uniform(-1, 1, g.cells), p=rng.uniform(-1, 1, g.faces),
                d=3.0 + rng.uniform(-1, 1, g.faces), o=rng.uniform(-1, 1, g.faces),
                y=rng.uniform(-1, 1, g.faces), ip=d.iplus, im=d.iminus)


@needs_ref
@pytest.mark.parametrize("gi", range(len(GRIDS)))
def test_oracle_bitwise_vs_reference(gi):
    g = GRIDS[gi]
    o, r = ffi.load("oracle"), ffi.load("ref")
    a = _inputs(g, 3 + gi)
    for fn, args in (("avg_x1", (a["b"],)), ("diff_x1", (a["b"],)), ("diff_x1_adjoint", (a["r"],)),
                     ("smoother_hessian_apply", (a["b"],)),
                     ("tridiag_apply", (a["d"], a["o"], a["p"], 0.75, a["y"])),
                     ("tridiag_solve_batched", (a["d"], a["o"], a["p"])),
                     ("dct_apply", (a["p"], 50.0, 1e3)),
                     ("distance_hessian_apply", (a["ip"], a["im"], a["b"], a["p"]))):
        assert np.array_equal(getattr(o, fn)(g, *args), getattr(r, fn)(g, *args)), fn
    assert o.is_strictly_feasible(g, a["b"]) == r.is_strictly_feasible(g, a["b"])
