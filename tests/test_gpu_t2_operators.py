"""The reference's test-side helpers of the hot path as
device entry points, bitwise against the oracle (itself pinned to the
reference in tests/test_t2_operators.py), host and device memory."""
import numpy as np
import pytest

from test_t2_operators import GRIDS, _inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gi", range(len(GRIDS)))
@pytest.mark.parametrize("on_device", [False, True])
def test_t2_bitwise_vs_oracle(ctx, oracle, gi, on_device):
    g = GRIDS[gi]
    a = _inputs(g, 3 + gi)
    if on_device:
        torch = pytest.importorskip("torch")
        dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in a.items()}
        host = lambda x: x.cpu().numpy()
    else:
        dev, host = a, (lambda x: x)
    for fn, keys, extra in (("avg_x1", ("b",), ()), ("diff_x1", ("b",), ()),
                            ("diff_x1_adjoint", ("r",), ()),
                            ("smoother_hessian_apply", ("b",), ()),
                            ("dct_apply", ("p",), (50.0, 1e3)),
                            ("distance_hessian_apply", ("ip", "im", "b", "p"), ()),
                            ("tridiag_solve_batched", ("d", "o", "p"), ())):
        got = getattr(ctx, fn)(g, *[dev[k] for k in keys], *extra)
        want = getattr(oracle, fn)(g, *[a[k] for k in keys], *extra)
        assert np.array_equal(host(got), want), fn
    got = ctx.tridiag_apply(g, dev["d"], dev["o"], dev["p"], 0.75, dev["y"])
    assert np.array_equal(host(got), oracle.tridiag_apply(g, a["d"], a["o"], a["p"], 0.75, a["y"]))
    assert ctx.is_strictly_feasible(g, dev["b"]) == oracle.is_strictly_feasible(g, a["b"])


def test_t2_tridiag_pivot_error_names_column(ctx):
    g = GRIDS[3]
    bad = np.ones(g.faces)
    bad[1 * g.n1 + 1] = -2.0
    with pytest.raises(RuntimeError, match="column 1"):
        ctx.tridiag_solve_batched(g, bad, np.zeros(g.faces), np.ones(g.faces))
    assert not ctx.is_strictly_feasible(g, np.arange(g.faces, dtype=np.float64) * 2.0)
