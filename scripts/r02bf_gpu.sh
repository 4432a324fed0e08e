#!/bin/bash
# which part of the tail-help change costs the main path (C3 b-step, 100 iterations)
O=gpurun_out
mkdir -p $O
for r in 1 2; do
for V in base none nohl nocoop cur; do
  if [ $V = cur ]; then L="EPC_BSTEP_HELP=1"; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bf_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "admm_bstep" $O/r02bf_c3_$V.log)"
done
done
