#!/bin/bash
# tail help v3 (helpers as a second kernel on a second stream): A/B + bitwise tests
O=gpurun_out
mkdir -p $O
sel() { case $1 in base) echo EPC_LIB=scripts/_var/base.so;; nohl2) echo EPC_LIB=scripts/_var/nohl2.so;; h0) echo EPC_BSTEP_HELP=0;; *) echo EPC_BSTEP_HELP=1;; esac; }
for r in 1 2; do
for V in base h1 h0 nohl2; do
  env $(sel $V) timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bg_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "admm_bstep" $O/r02bg_c3_$V.log)"
done
done
for V in base h1 h0; do
  env $(sel $V) timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02bg_x400_$V.log 2>&1
  echo "$V x400: $(grep -E "admm_bstep" $O/r02bg_x400_$V.log)"
done
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py -q -x > $O/r02bg_tests.log 2>&1
tail -2 $O/r02bg_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or x400" > $O/r02bg_full.log 2>&1
tail -2 $O/r02bg_full.log
