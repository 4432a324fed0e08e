#!/bin/bash
# heavy-column probe with per-column QP sub-phases and factor counters
O=gpurun_out
mkdir -p $O
export EPC_LIB=scripts/_var/heavy.so
timeout 300 python scripts/probe_heavy.py C3 1.0 60 10 > $O/r02bc_heavy_c3_60.log 2>&1
timeout 300 python scripts/probe_heavy.py C3 1.0 30 5 > $O/r02bc_heavy_c3_30.log 2>&1
timeout 300 python scripts/probe_heavy.py C3 400.0 40 3 > $O/r02bc_heavy_x400_40.log 2>&1
cat $O/r02bc_heavy_*.log
