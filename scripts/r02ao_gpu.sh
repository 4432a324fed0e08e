#!/bin/bash
# b-step column staging: EPC_STAGE_UNROLL 1 / 3 / 9 (C3 and x400 b-step time)
O=gpurun_out
for i in 1 2; do
for V in base stage3 stage9; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02ao_c3_${V}_$i.log 2>&1
  echo "$V $i: $(grep admm_bstep $O/r02ao_c3_${V}_$i.log)"
done
done
