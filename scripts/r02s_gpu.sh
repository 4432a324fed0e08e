#!/bin/bash
# PCG update kernel: memory-only / sweep-only timing split (C3)
O=gpurun_out
for V in base pcgnosweep pcgnomem; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  for i in 1 2; do
    env $L timeout 300 python scripts/probe_pcg.py C3 > $O/r02s_pcg_${V}_$i.log 2>&1
    echo "$V $i: $(grep block $O/r02s_pcg_${V}_$i.log)"
  done
done
