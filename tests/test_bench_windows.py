"""bench.py's reference arm times the whole solve as consecutive windows,
each warm-started from the previous window's state (ADMMState init,
admm.hpp:127-129; GN from the previous b). That must be the very same
trajectory as one uninterrupted call: checked here on the C port, which is
bitwise the reference (tests/test_oracle_pin.py)."""
import numpy as np

import bench
from paper_1607_00531_b200 import abi, synth


def test_admm_windows_continue_the_trajectory(oracle):
    d = synth.make_pair(synth.SynthSpec(m=(20, 12, 8), seed=3))
    full = oracle.admm_solve(d.grid, d.iplus, d.iminus, cfg=bench.admm_cfg(23))
    state = None
    rows = []
    bounds = bench.window_sizes(23, 5)
    for s in range(5):
        _, _, state = bench.ref_admm_window(oracle, 1, d, state, bounds[s + 1] - bounds[s])
        rows += state["rows"]
    for k in ("b", "z", "u"):
        assert np.array_equal(state[k], full[k]), k
    assert state["rho"] == full["rho"]
    assert [r["rho"] for r in rows] == [r["rho"] for r in full["rows"]]
    assert bench.window_sizes(100, 20) == list(range(0, 101, 5))
    assert bench.window_sizes(3, 5) is None


def test_gn_windows_continue_the_trajectory(oracle):
    d = synth.make_pair(synth.SynthSpec(m=(16, 12, 8), seed=4))
    cfg = bench.gn_config()
    cfg.max_outer = 4
    full = oracle.gn_solve(d.grid, d.iplus, d.iminus, cfg=cfg)
    b = None
    cfg1 = bench.gn_config()
    cfg1.max_outer = 1
    for _ in range(4):
        r = oracle.gn_solve(d.grid, d.iplus, d.iminus, b0=b, cfg=cfg1)
        b = r["b"]
    assert np.array_equal(b, full["b"])
