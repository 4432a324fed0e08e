#!/bin/bash
O=gpurun_out
for i in 1 2; do
for V in hvpm4 hvpm5 hvpm6 hvpm8; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_pcg.py C3 > $O/r02af_pcg_${V}_$i.log 2>&1
  echo "$V $i: $(grep block $O/r02af_pcg_${V}_$i.log)"
done
done
