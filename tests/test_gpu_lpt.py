"""Longest-columns-first claim order of the b-step (api.cu: EPC_LPT_MIN_MS).

By default only launches following a b-step of 5 ms or more are reordered, which
the small parity grids never reach. Here the switch is forced to "every launch"
in a child process (it is read once per process) and the bitwise ADMM parity
cases run again: single solves at x1 / x400 (admm.cpp:488-560), long columns,
and the batch entry with pairs stopping at different iterations and a failing
column, each against the oracle exactly as in the default order."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = ["tests/test_gpu_admm.py::test_admm_solve_small_bitwise",
         "tests/test_gpu_admm.py::test_admm_solve_long_columns_bitwise",
         "tests/test_gpu_admm.py::test_admm_solve_default_tolerances_stop_early",
         "tests/test_gpu_fullsize.py::test_admm_batch_pairs_each_bitwise",
         "tests/test_gpu_fullsize.py::test_admm_batch_warm_start_fixed_count",
         "tests/test_gpu_admm_loop.py::test_pipelined_batch_matches_sync_loop"]


@pytest.mark.gpu
@pytest.mark.parametrize("two", ["0", "1"])
def test_parity_cases_with_every_launch_reordered(two):
    env = dict(os.environ, EPC_LPT_MIN_MS="0", EPC_LPT_TWO=two)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", *CASES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
