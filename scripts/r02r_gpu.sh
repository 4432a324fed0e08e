#!/bin/bash
set -x
O=gpurun_out
EPC_BSTEP_PAIR=1 timeout 900 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_dist.py tests/test_gpu_multilevel.py -q -x > $O/r02r_tests_pair.log 2>&1
tail -3 $O/r02r_tests_pair.log
for i in 1 2; do
for V in 0 1; do
  EPC_BSTEP_PAIR=$V timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02r_c3_pair${V}_$i.log 2>&1
done
EPC_LIB=scripts/_var/r1.so python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02r_c3_r1_$i.log 2>&1
done
EPC_BSTEP_PAIR=1 timeout 300 python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02r_x400_pair1.log 2>&1
EPC_BSTEP_PAIR=0 timeout 300 python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02r_x400_pair0.log 2>&1
EPC_BSTEP_PAIR=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or x400" > $O/r02r_fullsize_pair.log 2>&1
for f in $O/r02r_c3_*.log $O/r02r_x400_*.log; do echo "$f $(grep admm_bstep $f | awk '{print $2}')"; done
tail -3 $O/r02r_fullsize_pair.log
