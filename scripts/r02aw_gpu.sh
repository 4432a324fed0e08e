#!/bin/bash
# b-step occupancy: 8 warps/SM at 252 registers vs 9-10 at 168 (spills), images staged or via L1
O=gpurun_out
for cfg in "base:" "base:EPC_BSTEP_IMG=1" "m9:" "m12:EPC_BSTEP_IMG=1"; do
  V=${cfg%%:*}; E=${cfg#*:}
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L $E timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02aw.log 2>&1
  echo "$V $E C3: $(grep -E "admm_bstep" $O/r02aw.log)"
  env $L $E timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02aw.log 2>&1
  echo "$V $E x400: $(grep -E "admm_bstep" $O/r02aw.log)"
done
