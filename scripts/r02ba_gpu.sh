#!/bin/bash
# b-step segmented chains: warm-up of 0 / 1 / 2 / 3 segments before each lane's segment
O=gpurun_out
EPC_LIB=scripts/_var/w3.so timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py -q -x > $O/r02ba_tests.log 2>&1
tail -2 $O/r02ba_tests.log
for V in base w1 w2 w3; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02ba.log 2>&1
  echo "$V C3: $(grep -E "admm_bstep" $O/r02ba.log)"
  env $L timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02ba.log 2>&1
  echo "$V x400: $(grep -E "admm_bstep" $O/r02ba.log)"
done
