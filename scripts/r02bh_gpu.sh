#!/bin/bash
# main-path cost of the tail-help hooks with help off (C3 b-step, 100 iterations)
O=gpurun_out
mkdir -p $O
for r in 1 2; do
for V in base h0 nodone noowner; do
  case $V in base|nodone|noowner) L="EPC_LIB=scripts/_var/$V.so EPC_BSTEP_HELP=0";; h0) L="EPC_BSTEP_HELP=0";; esac
  env $L timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bh_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "admm_bstep" $O/r02bh_c3_$V.log)"
done
done
