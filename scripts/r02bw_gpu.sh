#!/bin/bash
# cell index + 0.5 carried as a double in the trial and model loops: A/B + bitwise tests
O=gpurun_out
mkdir -p $O
sel() { case $1 in cur) echo "EPC_BSTEP_X=1";; *) echo "EPC_LIB=scripts/_var/$1.so";; esac; }
for r in 1 2; do
for V in base cur; do
  env $(sel $V) timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bw_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "admm_bstep" $O/r02bw_c3_$V.log)"
done
done
for V in base cur; do
  env $(sel $V) timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02bw_x400_$V.log 2>&1
  echo "$V x400: $(grep -E "admm_bstep" $O/r02bw_x400_$V.log)"
done
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py -q -x > $O/r02bw_tests.log 2>&1
tail -2 $O/r02bw_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or x400" > $O/r02bw_full.log 2>&1
tail -2 $O/r02bw_full.log
