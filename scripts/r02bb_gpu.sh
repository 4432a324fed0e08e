#!/bin/bash
# heavy-column probe (C3 late / early, x400 late) + GN GPU tests at HEAD
O=gpurun_out
mkdir -p $O
export EPC_LIB=scripts/_var/heavy.so
timeout 300 python scripts/probe_heavy.py C3 1.0 60 10 > $O/r02bb_heavy_c3_60.log 2>&1
timeout 300 python scripts/probe_heavy.py C3 1.0 10 5 > $O/r02bb_heavy_c3_10.log 2>&1
timeout 300 python scripts/probe_heavy.py C3 400.0 40 3 > $O/r02bb_heavy_x400_40.log 2>&1
unset EPC_LIB
timeout 900 python -m pytest tests/test_gpu_gn.py -x -q -m gpu > $O/r02bb_gn_tests.log 2>&1
cat $O/r02bb_heavy_*.log; tail -3 $O/r02bb_gn_tests.log
