#!/bin/bash
# PCG update: multiply-high column index, unrolled segments (A/B)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02v_tests_gn.log 2>&1
tail -2 $O/r02v_tests_gn.log
for i in 1 2; do
for V in base nounr pcgold; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_pcg.py C3 > $O/r02v_pcg_${V}_$i.log 2>&1
  echo "$V $i: $(grep block $O/r02v_pcg_${V}_$i.log)"
done
done
for V in base pcgold; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  for C in C2 C3; do
    env $L timeout 300 python scripts/probe_gn.py --config $C > $O/r02v_gn_${V}_$C.log 2>&1
    echo "$V $C: $(grep -E "^GN|pcg_update|pcg_loop" $O/r02v_gn_${V}_$C.log | tr "\n" " ")"
  done
done
