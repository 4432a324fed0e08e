#!/bin/bash
# GN C2 (configs[1]): loop vs per-iteration kernels, 16 vs 8 columns per block (warm-up segments)
O=gpurun_out
for cfg in "" "EPC_PCG_CPW=8" "EPC_PCG_LOOP=0" "EPC_PCG_LOOP=0 EPC_PCG_CPW=8"; do
  env $cfg timeout 300 python scripts/probe_gn.py --config C2 > $O/r02al.log 2>&1
  echo "[$cfg] $(grep -E "^GN" $O/r02al.log)"
  grep -E "pcg_loop|pcg_update|pcg_hvp" $O/r02al.log
done
