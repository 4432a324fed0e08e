#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02ad_tests_gn.log 2>&1
tail -2 $O/r02ad_tests_gn.log
for i in 1 2; do
for V in base segwarm0; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  for C in C2 C3; do
    env $L timeout 300 python scripts/probe_gn.py --config $C > $O/r02ad_gn_${V}_${C}_$i.log 2>&1
    echo "$V $C $i: $(grep -E "^GN|pcg_update|pcg_loop" $O/r02ad_gn_${V}_${C}_$i.log | tr "\n" " ")"
  done
done
done
