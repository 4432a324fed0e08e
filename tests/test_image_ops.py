"""correct_pair / ssd / ncc / simulate_pair (
proj/src/image.cpp) on CPU: the oracle restatement bitwise against the live
reference library (including simulate_pair's mt19937_64 / normal_distribution
noise stream), and the reference's error behaviour. GPU: test_gpu_image_ops.py."""
import numpy as np
import pytest

from kats import phantom_gaussian
from oracle import ffi
from paper_1607_00531_b200 import abi, synth

needs_ref = pytest.mark.skipif(not ffi.available("ref"), reason="reference library not available")


def case(m=(20, 14, 6), seed=3, amp=0.6):
    d = synth.make_pair(synth.SynthSpec(m=m, seed=seed, d1_max=amp))
    return d


@needs_ref
@pytest.mark.parametrize("m", [(20, 14, 6), (17, 9, 1), (33, 12, 5)])
def test_oracle_image_ops_bitwise_vs_reference(m):
    orc, ref = ffi.load("oracle"), ffi.load("ref")
    d = case(m)
    g = d.grid
    b = d.b_true if d.b_true is not None else np.zeros(g.faces)
    a1, a2 = orc.correct_pair(g, d.iplus, d.iminus, b), ref.correct_pair(g, d.iplus, d.iminus, b)
    assert np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1])
    assert orc.ssd(g, a1[0], a1[1]) == ref.ssd(g, a1[0], a1[1])
    assert orc.ncc(g, a1[0], a1[1]) == ref.ncc(g, a1[0], a1[1])
    truth = phantom_gaussian(g)
    for sigma, seed in ((0.0, 0), (0.01, 7), (0.3, 12345)):
        s1 = orc.simulate_pair(g, truth, b, sigma, seed)
        s2 = ref.simulate_pair(g, truth, b, sigma, seed)
        assert np.array_equal(s1[0], s2[0]) and np.array_equal(s1[1], s2[1]), sigma


@pytest.mark.parametrize("kind", ["oracle", "ref"])
def test_image_ops_errors(kind):
    if kind == "ref" and not ffi.available("ref"):
        pytest.skip("reference library not available")
    c = ffi.load(kind)
    g = abi.Grid.make(8, 6, 1)
    steep = np.tile(np.arange(9) * 1.2, 6)   # |D1 b| = 1.2
    with pytest.raises(ValueError, match="correct_pair: field infeasible"):
        c.correct_pair(g, np.ones(g.cells), np.ones(g.cells), steep)
    with pytest.raises(ValueError, match="simulate_pair: field infeasible, max"):
        c.simulate_pair(g, np.ones(g.cells), np.tile(np.arange(9) * 0.97, 6))
    with pytest.raises(ValueError, match="ncc: zero-variance image"):
        c.ncc(g, np.ones(g.cells), np.arange(g.cells, dtype=float))
