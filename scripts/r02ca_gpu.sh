#!/bin/bash
# fp32 dual kernel with 32-bit index arithmetic: A/B + fp32 tests
O=gpurun_out
mkdir -p $O
sel() { case $1 in cur) echo "EPC_BSTEP_X=1";; *) echo "EPC_LIB=scripts/_var/$1.so";; esac; }
for r in 1 2; do
for V in base cur; do
  env $(sel $V) timeout 300 python scripts/probe_f32_time.py C3 100 > $O/r02ca_f32_$V.log 2>&1
  echo "$V: $(head -1 $O/r02ca_f32_$V.log) $(grep -E "bstep|dual" $O/r02ca_f32_$V.log)"
done
done
timeout 1200 python -m pytest tests/test_gpu_admm_f32.py -q -x > $O/r02ca_tests.log 2>&1
tail -2 $O/r02ca_tests.log
