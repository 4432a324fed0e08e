#!/bin/bash
set -x
O=gpurun_out
for i in 1 2; do
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02l_c3_now$i.log 2>&1
EPC_LIB=scripts/_var/r1.so python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02l_c3_r1_$i.log 2>&1
done
python scripts/probe_gn.py --config C2 > $O/r02l_gn_c2.log 2>&1
EPC_LIB=scripts/_var/r1.so python scripts/probe_gn.py --config C2 > $O/r02l_gn_c2_r1.log 2>&1
python -m pytest tests/test_gpu_gn.py tests/test_gpu_admm.py -q > $O/r02l_tests.log 2>&1
grep -h "admm 100\|admm_bstep\|unprofiled" $O/r02l_*.log
