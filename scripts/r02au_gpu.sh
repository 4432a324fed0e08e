#!/bin/bash
# interpolant end ramps behind a branch (EPC_INTERP_EDGE_BRANCH): bitwise tests, C3 / x400 b-step time
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py tests/test_gpu_gn.py tests/test_gpu_image.py -q -x > $O/r02au_tests.log 2>&1
tail -2 $O/r02au_tests.log
for V in base edge0; do
  if [ $V = base ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02au_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "^admm|admm_bstep" $O/r02au_c3_$V.log | tr '\n' ' ')"
  env $L timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02au_x400_$V.log 2>&1
  echo "$V x400: $(grep -E "admm_bstep" $O/r02au_x400_$V.log)"
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or x400" > $O/r02au_full.log 2>&1
tail -2 $O/r02au_full.log
