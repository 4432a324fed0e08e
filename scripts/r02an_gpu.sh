#!/bin/bash
# ncu source-level capture of the C2 persistent PCG loop (probe_gn --ncu exited 0 before)
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pcg_loop -c 1 \
  -o $O/r02an_loop_c2 -f python scripts/probe_gn.py --config C2 --ncu > $O/r02an_ncu.log 2>&1
tail -2 $O/r02an_ncu.log
