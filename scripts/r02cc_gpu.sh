#!/bin/bash
# 48-row tiles for the forward axis-3 divide GEMM: A/B + tests
O=gpurun_out
mkdir -p $O
sel() { case $1 in cur) echo "EPC_BSTEP_X=1";; *) echo "EPC_LIB=scripts/_var/$1.so";; esac; }
for r in 1 2; do
for V in base cur; do
  env $(sel $V) timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02cc_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "^admm" $O/r02cc_c3_$V.log) $(grep -E "dct" $O/r02cc_c3_$V.log | tr '\n' ' ')"
done
done
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py tests/test_gpu_dist.py tests/test_gpu_t2_operators.py tests/test_gpu_multilevel.py -q -x > $O/r02cc_tests.log 2>&1
tail -2 $O/r02cc_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or batch" > $O/r02cc_full.log 2>&1
tail -2 $O/r02cc_full.log
