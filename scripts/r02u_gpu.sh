#!/bin/bash
# PCG update: register-held segmented sweeps with warp-local divisions (A/B)
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02u_tests_gn.log 2>&1
tail -2 $O/r02u_tests_gn.log
for i in 1 2; do
for V in base segwarp0 dvahead; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_pcg.py C3 > $O/r02u_pcg_${V}_$i.log 2>&1
  echo "$V $i: $(grep block $O/r02u_pcg_${V}_$i.log)"
done
done
for V in base segwarp0; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  for C in C2 C3; do
    env $L timeout 300 python scripts/probe_gn.py --config $C > $O/r02u_gn_${V}_$C.log 2>&1
    echo "$V $C: $(grep -E "^GN|pcg_update" $O/r02u_gn_${V}_$C.log | tr "\n" " ")"
  done
done
