"""GN-PCG hot path on the GPU vs the oracle (bitwise-pinned C restatement of
the reference). Element-wise pieces (gradient, residual, Hessian blocks,
stencil apply, preconditioners) must be bitwise; scalars that the reference
reduces sequentially are fixed-order tree sums here (rel 1e-12); whole
solves are held to the north-star tolerance (b rel L2 <= 1e-8, j_value rel
<= 1e-9 at fixed iteration counts)."""
import numpy as np
import pytest

from paper_1607_00531_b200 import abi, synth

pytestmark = pytest.mark.gpu


def pair(m=(16, 12, 8), seed=9, scale=1.0):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=seed))
    return d.grid, d.iplus * scale, d.iminus * scale, d.b_true


def field(g, rng, amp=0.3):
    b = rng.uniform(-1, 1, g.faces)
    # keep |D1 b| well inside 1
    bb = b.reshape(-1, g.n1)
    bb[:] = np.cumsum(amp * 0.5 * rng.uniform(-1, 1, bb.shape), axis=1)
    return np.ascontiguousarray(bb.ravel())


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_objective_gn(ctx, oracle, scale):
    g, ip, im, _ = pair(scale=scale)
    rng = np.random.default_rng(1)
    for b in (np.zeros(g.faces), field(g, rng)):
        for need_grad in (True, False):
            r = oracle.objective_gn(g, ip, im, b, need_grad=need_grad)
            o = ctx.objective_gn(g, ip, im, b, need_grad=need_grad)
            assert o["feasible"] == r["feasible"]
            for k in ("value", "dist", "smooth", "pen"):
                assert o[k] == pytest.approx(r[k], rel=1e-12, abs=1e-300), k
            if need_grad:
                assert np.array_equal(o["grad"], r["grad"])
                assert np.array_equal(o["residual"], r["residual"])


def test_objective_infeasible(ctx, oracle):
    g, ip, im, _ = pair()
    b = np.zeros(g.faces)
    b.reshape(-1, g.n1)[:, 3] = 2.0  # |D1 b| = 2
    o = ctx.objective_gn(g, ip, im, b)
    r = oracle.objective_gn(g, ip, im, b)
    assert not o["feasible"] and not r["feasible"]
    assert o["value"] == np.inf == r["value"]


def test_hessian_blocks_and_apply_bitwise(ctx, oracle):
    g, ip, im, _ = pair(scale=400.0)
    rng = np.random.default_rng(2)
    b = field(g, rng)
    r = oracle.gn_hessian_build(g, ip, im, b)
    o = ctx.gn_hessian_build(g, ip, im, b)
    for k in ("diag", "off", "pdiag"):
        assert np.array_equal(o[k], r[k]), k
    x = rng.uniform(-1, 1, g.faces)
    assert np.array_equal(ctx.gn_hessian_apply(g, ip, im, b, x), oracle.gn_hessian_apply(g, ip, im, b, x))


@pytest.mark.parametrize("kind", [abi.PRECOND_NONE, abi.PRECOND_JACOBI, abi.PRECOND_BLOCK_JACOBI])
def test_preconditioners_bitwise(ctx, oracle, kind):
    g, ip, im, _ = pair(scale=400.0)
    rng = np.random.default_rng(3)
    b = field(g, rng)
    rr = rng.uniform(-1, 1, g.faces)
    assert np.array_equal(ctx.precond_apply(g, ip, im, b, kind, rr),
                          oracle.precond_apply(g, ip, im, b, kind, rr))


@pytest.mark.parametrize("kind", [abi.PRECOND_JACOBI, abi.PRECOND_BLOCK_JACOBI])
def test_pcg(ctx, oracle, kind):
    g, ip, im, _ = pair(scale=400.0)
    rng = np.random.default_rng(4)
    b = field(g, rng)
    grad = oracle.objective_gn(g, ip, im, b)["grad"]
    r = oracle.pcg(g, ip, im, b, grad, 1e-2, 50, kind=kind)
    o = ctx.pcg(g, ip, im, b, grad, 1e-2, 50, kind=kind)
    assert o["iters"] == r["iters"]
    assert o["reached_tol"] == r["reached_tol"]
    assert o["relres"] == pytest.approx(r["relres"], rel=1e-9)
    rel = np.linalg.norm(o["d"] - r["d"]) / np.linalg.norm(r["d"])
    assert rel <= 1e-10


@pytest.mark.parametrize("m", [(16, 7, 3), (15, 9, 1), (299, 5, 3)])
@pytest.mark.parametrize("path", [{}, {"EPC_PCG_LOOP": "0"}, {"EPC_PCG_CPW": "0"}])
def test_pcg_block_ragged_shapes(ctx, oracle, monkeypatch, m, path):
    """Block-Jacobi PCG on shapes that exercise the kernels' edges: a last
    column group with fewer than CPW columns and an odd face count (the
    16-byte passes then finish with a scalar face), a 2D grid (no k
    neighbours) and long columns (8 columns per block). Each of the three
    device paths (persistent loop, per-iteration launches, warp-per-column
    kernel) must match the oracle."""
    for k, v in path.items():
        monkeypatch.setenv(k, v)
    g, ip, im, _ = pair(m=m, scale=400.0)
    rng = np.random.default_rng(5)
    b = field(g, rng)
    grad = oracle.objective_gn(g, ip, im, b)["grad"]
    r = oracle.pcg(g, ip, im, b, grad, 1e-3, 40, kind=abi.PRECOND_BLOCK_JACOBI)
    o = ctx.pcg(g, ip, im, b, grad, 1e-3, 40, kind=abi.PRECOND_BLOCK_JACOBI)
    assert o["iters"] == r["iters"] and o["reached_tol"] == r["reached_tol"]
    assert o["relres"] == pytest.approx(r["relres"], rel=1e-9)
    assert np.linalg.norm(o["d"] - r["d"]) / np.linalg.norm(r["d"]) <= 1e-10


def test_pcg_zero_gradient(ctx, oracle):
    g, ip, im, _ = pair()
    o = ctx.pcg(g, ip, im, np.zeros(g.faces), np.zeros(g.faces), 0.1, 10)
    assert o["iters"] == 0 and o["reached_tol"] and not o["d"].any()


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_gn_solve_small(ctx, oracle, scale):
    g, ip, im, _ = pair(m=(20, 16, 10), scale=scale)
    cfg = abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=10)
    r = oracle.gn_solve(g, ip, im, cfg=cfg)
    o = ctx.gn_solve(g, ip, im, cfg=cfg)
    assert o["stop"] == r["stop"] and len(o["rows"]) == len(r["rows"])
    rel = np.linalg.norm(o["b"] - r["b"]) / np.linalg.norm(r["b"])
    assert rel <= 1e-8, rel
    for a, b in zip(o["rows"], r["rows"]):
        assert a["pcg_iters"] == b["pcg_iters"]
        assert a["step"] == b["step"]
        assert a["j_value"] == pytest.approx(b["j_value"], rel=1e-9)
        assert a["grad_norm"] == pytest.approx(b["grad_norm"], rel=1e-7)


def test_gn_identical_images_stop_immediately(ctx, oracle):
    g, ip, _, _ = pair()
    o = ctx.gn_solve(g, ip, ip.copy())
    r = oracle.gn_solve(g, ip, ip.copy())
    assert o["stop"] == r["stop"]
    assert o["message"] == r["message"]


def test_gn_infeasible_start_raises(ctx):
    g, ip, im, _ = pair()
    b0 = np.zeros(g.faces)
    b0.reshape(-1, g.n1)[:, 2] = 5.0
    with pytest.raises(ValueError, match="starting guess is infeasible"):
        ctx.gn_solve(g, ip, im, b0=b0)


@pytest.mark.slow
def test_gn_c2_parity(ctx, oracle):
    d = synth.make_config("C2")
    cfg = abi.GnConfig(eta=1e-2, max_pcg=50, max_outer=10)
    r = oracle.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    o = ctx.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    rel = np.linalg.norm(o["b"] - r["b"]) / np.linalg.norm(r["b"])
    assert rel <= 1e-8, rel
    for a, b in zip(o["rows"], r["rows"]):
        assert a["pcg_iters"] == b["pcg_iters"]
        assert a["j_value"] == pytest.approx(b["j_value"], rel=1e-9)


@pytest.mark.parametrize("m", [(128, 9, 5), (256, 7, 3), (300, 5, 3), (512, 5, 2), (16, 7, 3)])
@pytest.mark.parametrize("loop", ["1", "0"])
def test_pcg_segmented_sweeps_bitwise(ctx, oracle, monkeypatch, m, loop):
    """The block-Jacobi sweeps as warp-per-column segmented chains (pcg.cu
    sweeps_seg: segments of 9 / 17 steps with agreement rounds, 8 columns
    per block) return the very bits of the thread-per-column chains
    (EPC_PCG_SEG=0): d, the iteration count and relres identical, on column
    lengths n1 = 257, 301 and 513 (n1 = 129 and a short column keep the
    thread chains at 16 columns per block: both settings run the same code),
    in the persistent loop and in the per-iteration kernels."""
    monkeypatch.setenv("EPC_PCG_LOOP", loop)
    g, ip, im, _ = pair(m=m, scale=400.0)
    rng = np.random.default_rng(8)
    b = field(g, rng)
    grad = oracle.objective_gn(g, ip, im, b)["grad"]
    seg = ctx.pcg(g, ip, im, b, grad, 1e-4, 30, kind=abi.PRECOND_BLOCK_JACOBI)
    monkeypatch.setenv("EPC_PCG_SEG", "0")
    one = ctx.pcg(g, ip, im, b, grad, 1e-4, 30, kind=abi.PRECOND_BLOCK_JACOBI)
    assert np.array_equal(seg["d"], one["d"])
    assert seg["iters"] == one["iters"] and seg["relres"] == one["relres"]
    r = oracle.pcg(g, ip, im, b, grad, 1e-4, 30, kind=abi.PRECOND_BLOCK_JACOBI)
    assert seg["iters"] == r["iters"]
    assert np.linalg.norm(seg["d"] - r["d"]) / np.linalg.norm(r["d"]) <= 1e-10


@pytest.mark.parametrize("m,h", [((16, 12, 8), (1.0, 1.0, 1.0)), ((15, 9, 1), (0.8, 1.3, 1.0)),
                                 ((12, 7, 5), (1.0, 0.7, 1.6))])
def test_gn_operators_from_column_blocks(ctx, oracle, m, h):
    """The C ABI behind the shim's GnHessian / make_preconditioner: the
    stencil apply from the column part (GnHessian::apply), the
    preconditioner-block diagonal (= full_diagonal()), the Jacobi apply and
    the block-Jacobi apply (tridiag_solve_batched on the preconditioner
    blocks), each bitwise against the oracle's own GnHessian pieces."""
    d0 = synth.make_pair(synth.SynthSpec(m=m, seed=12))
    g = abi.Grid.make(*m, h=h)
    ip, im = d0.iplus * 400.0, d0.iminus * 400.0
    rng = np.random.default_rng(3)
    b = field(g, rng)
    x = rng.uniform(-1, 1, g.faces)
    params = abi.ObjectiveParams()
    hb = oracle.gn_hessian_build(g, ip, im, b, params=params)
    V = h[0] * h[1] * h[2]
    w2 = params.alpha * V / (h[1] * h[1])
    w3 = params.alpha * V / (h[2] * h[2]) if m[2] > 1 else 0.0
    y = ctx.gn_stencil_apply(g, hb["diag"], hb["off"], w2, w3, x)
    assert np.array_equal(y, oracle.gn_hessian_apply(g, ip, im, b, x, params=params))
    pd = ctx.gn_cross_diag_add(g, hb["diag"], w2, w3)
    assert np.array_equal(pd, hb["pdiag"])
    r = rng.uniform(-1, 1, g.faces)
    zj = ctx.jacobi_apply(pd, r)
    assert np.array_equal(zj, oracle.precond_apply(g, ip, im, b, abi.PRECOND_JACOBI, r, params=params))
    zb = ctx.tridiag_solve_batched(g, pd, hb["off"], r)
    assert np.array_equal(zb, oracle.precond_apply(g, ip, im, b, abi.PRECOND_BLOCK_JACOBI, r,
                                                   params=params))
