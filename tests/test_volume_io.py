"""Volume files (proj/src/volume_io.cpp): the product's
host-side epc_write_volume / epc_read_volume against the reference library -
byte-identical files, cross-reading both ways - and its own round trip.
The device permutations are in test_gpu_volume_io.py."""
import numpy as np
import pytest

from oracle import ffi
from paper_1607_00531_b200 import abi, epicorr

needs_ref = pytest.mark.skipif(not ffi.available("ref"), reason="reference library not available")
CASES = [(abi.Grid.make(6, 5, 4, h=(1.0, 0.7, 1.3), origin=(0.1, -2.0, 3.5)), 0),
         (abi.Grid.make(6, 5, 4), 1), (abi.Grid.make(6, 5, 4), 2), (abi.Grid.make(6, 5, 4), 3),
         (abi.Grid.make(7, 3, 1, h=(0.5, 2.0, 1.0)), 0), (abi.Grid.make(7, 3, 1), 1)]


def payload(g, kind, seed=1):
    pd = list(g.m)
    if kind:
        pd[kind - 1] += 1
    return np.random.default_rng(seed).normal(size=pd[0] * pd[1] * pd[2])


@pytest.mark.parametrize("g,kind", CASES)
def test_product_round_trip(tmp_path, g, kind):
    v = payload(g, kind)
    p = tmp_path / "a.vol"
    epicorr.write_volume(p, g, kind, v)
    g2, k2, v2 = epicorr.read_volume(p)
    assert k2 == kind and list(g2.m) == list(g.m) and list(g2.h) == list(g.h)
    assert list(g2.origin) == list(g.origin)
    assert np.array_equal(v2, v.astype(np.float32).astype(np.float64))


@needs_ref
@pytest.mark.parametrize("g,kind", CASES)
def test_files_match_reference(tmp_path, g, kind):
    ref = ffi.load("ref")
    v = payload(g, kind)
    a, b = tmp_path / "ours.vol", tmp_path / "ref.vol"
    epicorr.write_volume(a, g, kind, v)
    ref.write_volume(str(b), g, kind, v)
    assert a.read_bytes() == b.read_bytes()
    g1, k1, v1 = ref.read_volume(str(a))
    g2, k2, v2 = epicorr.read_volume(b)
    assert k1 == k2 == kind and np.array_equal(v1, v2)
    for x, y in ((g1, g2), (g1, g)):
        assert list(x.m) == list(y.m) and list(x.h) == list(y.h) and list(x.origin) == list(y.origin)
