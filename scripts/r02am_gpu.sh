#!/bin/bash
# GN C2: half-warp segmented sweeps at 16 columns per block (EPC_PCG_SEG16) - bitwise + timing
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02am_tests.log 2>&1
tail -2 $O/r02am_tests.log
for i in 1 2; do
for cfg in "EPC_PCG_SEG16=1" "EPC_PCG_SEG16=0" "EPC_PCG_LOOP=0 EPC_PCG_SEG16=1" "EPC_PCG_LOOP=0 EPC_PCG_SEG16=0"; do
  env $cfg timeout 300 python scripts/probe_gn.py --config C2 > $O/r02am.log 2>&1
  echo "[$cfg] $(grep -E "^GN" $O/r02am.log) $(grep -E "pcg_loop|pcg_update" $O/r02am.log | tr '\n' ' ')"
done
done
