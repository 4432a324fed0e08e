#!/bin/bash
# full GPU suite after the PCG update / hvp changes, plus the C3 GN probe
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r02ag_tests_gpu.log 2>&1
tail -3 $O/r02ag_tests_gpu.log
timeout 300 python scripts/probe_gn.py --config C3 > $O/r02ag_gn_C3.log 2>&1
grep -E "^GN|pcg_update|pcg_hvp" $O/r02ag_gn_C3.log
