"""permute_to_axis1 / unpermute_field on the device against the reference
library (volume_io.cpp:203-223), bitwise, and their involution property."""
import numpy as np
import pytest

from oracle import ffi
from paper_1607_00531_b200 import abi

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ffi.available("ref"), reason="reference library not available")]


@pytest.mark.parametrize("g", [abi.Grid.make(6, 5, 4, h=(1.0, 0.7, 1.3)), abi.Grid.make(9, 4, 1)])
def test_permutations_match_reference(ctx, g):
    ref = ffi.load("ref")
    rng = np.random.default_rng(2)
    img, b = rng.normal(size=g.cells), rng.normal(size=g.faces)
    for pe in range(1, g.dim + 1):
        og, out = ctx.permute_to_axis1(g, pe, img)
        rg, rout = ref.permute_to_axis1(g, pe, img)
        assert np.array_equal(out, rout) and list(og.m) == list(rg.m) and list(og.h) == list(rg.h)
        back = ctx.permute_to_axis1(og, pe, out)[1]
        assert np.array_equal(back, img)
        og, kind, fo = ctx.unpermute_field(g, pe, b)
        rg, rk, rfo = ref.unpermute_field(g, pe, b)
        assert kind == rk and np.array_equal(fo, rfo) and list(og.m) == list(rg.m)
    with pytest.raises(ValueError):
        ctx.permute_to_axis1(g, g.dim + 1, img)
