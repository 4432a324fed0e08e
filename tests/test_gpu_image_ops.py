"""correct_pair / ssd / ncc / simulate_pair on the GPU against the oracle
(pinned bitwise to the reference by test_image_ops.py): correct_pair and
simulate_pair (noise included) bitwise; the metrics within rounding of their
fixed-order device sums."""
import numpy as np
import pytest
import torch

from kats import phantom_gaussian
from paper_1607_00531_b200 import abi, synth
from test_image_ops import case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m", [(20, 14, 6), (17, 9, 1), (64, 24, 8)])
def test_image_ops_match_reference(ctx, oracle, m):
    d = case(m)
    g = d.grid
    b = d.b_true
    got = ctx.correct_pair(g, d.iplus, d.iminus, b)
    ref = oracle.correct_pair(g, d.iplus, d.iminus, b)
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert ctx.ssd(g, got[0], got[1]) == pytest.approx(oracle.ssd(g, ref[0], ref[1]), rel=1e-12)
    assert ctx.ncc(g, got[0], got[1]) == pytest.approx(oracle.ncc(g, ref[0], ref[1]), rel=1e-12)
    truth = phantom_gaussian(g)
    for sigma, seed in ((0.0, 0), (0.01, 7)):
        s1 = ctx.simulate_pair(g, truth, b, sigma, seed)
        s2 = oracle.simulate_pair(g, truth, b, sigma, seed)
        assert np.array_equal(s1[0], s2[0]) and np.array_equal(s1[1], s2[1]), sigma
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(x).to(dev) for x in (d.iplus, d.iminus, b)]
    cpd = ctx.correct_pair(g, *t)
    assert np.array_equal(cpd[0].cpu().numpy(), ref[0])


def test_image_ops_errors_gpu(ctx):
    g = abi.Grid.make(8, 6, 1)
    with pytest.raises(ValueError, match="correct_pair: field infeasible"):
        ctx.correct_pair(g, np.ones(g.cells), np.ones(g.cells), np.tile(np.arange(9) * 1.2, 6))
    with pytest.raises(ValueError, match="simulate_pair: field infeasible, max"):
        ctx.simulate_pair(g, np.ones(g.cells), np.tile(np.arange(9) * 0.97, 6))
    with pytest.raises(ValueError, match="ncc: zero-variance image"):
        ctx.ncc(g, np.ones(g.cells), np.arange(g.cells, dtype=float))
