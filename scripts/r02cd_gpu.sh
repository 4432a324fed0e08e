#!/bin/bash
# 48-row tiles for the inverse axis-3 GEMM (variant rm3)
O=gpurun_out
mkdir -p $O
sel() { case $1 in cur) echo "EPC_BSTEP_X=1";; *) echo "EPC_LIB=scripts/_var/$1.so";; esac; }
for r in 1 2; do
for V in cur rm3; do
  env $(sel $V) timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02cd_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "^admm" $O/r02cd_c3_$V.log) $(grep -E "dct" $O/r02cd_c3_$V.log | tr '\n' ' ')"
done
done
