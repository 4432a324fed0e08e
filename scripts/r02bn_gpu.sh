#!/bin/bash
# DCT GEMM epilogues with 32-bit per-column index math (fp64 and fp32): A/B + tests
O=gpurun_out
mkdir -p $O
sel() { case $1 in cur) echo "EPC_BSTEP_X=1";; *) echo "EPC_LIB=scripts/_var/$1.so";; esac; }
for r in 1 2; do
for V in base cur; do
  env $(sel $V) timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bn_c3_$V.log 2>&1
  echo "$V C3: $(grep -E "^admm" $O/r02bn_c3_$V.log)"
  grep -E "dct|gemm" $O/r02bn_c3_$V.log
done
done
for V in base cur; do
  env $(sel $V) timeout 300 python scripts/probe_f32.py C3 100 > $O/r02bn_f32_$V.log 2>&1
  echo "$V f32:"; tail -12 $O/r02bn_f32_$V.log
done
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_f32.py tests/test_gpu_dist.py -q -x > $O/r02bn_tests.log 2>&1
tail -2 $O/r02bn_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full" > $O/r02bn_full.log 2>&1
tail -2 $O/r02bn_full.log
