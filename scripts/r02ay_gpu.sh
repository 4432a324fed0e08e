#!/bin/bash
# GN outer loop: deferred factor check + one read for the step's norms (fewer host round trips)
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gn.py tests/test_gpu_shim.py tests/test_gpu_fullsize.py -q -x -k "gn or GN or pcg or shim or objective or hessian or precond" > $O/r02ay_tests.log 2>&1
tail -2 $O/r02ay_tests.log
for i in 1 2; do
for V in base gnold; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_gn.py --config C2 > $O/r02ay.log 2>&1
  echo "$V C2: $(grep -E "^GN|unprofiled" $O/r02ay.log | tr '\n' ' ')"
done
done
