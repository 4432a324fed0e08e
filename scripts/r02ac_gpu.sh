#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02ac_tests_gn.log 2>&1
tail -2 $O/r02ac_tests_gn.log
for i in 1 2; do
for V in base warm0; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_pcg.py C3 > $O/r02ac_pcg_${V}_$i.log 2>&1
  echo "$V $i: $(grep block $O/r02ac_pcg_${V}_$i.log)"
done
done
