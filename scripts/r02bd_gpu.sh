#!/bin/bash
# tail help (cooperative line search in the b-step's tail): timing A/B and bitwise tests
O=gpurun_out
mkdir -p $O
for H in 1 0 1; do
  EPC_BSTEP_HELP=$H timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bd_c3_h$H.log 2>&1
  echo "help=$H C3: $(grep -E "^admm|admm_bstep" $O/r02bd_c3_h$H.log | tr '\n' ' ')"
done
for H in 1 0; do
  EPC_BSTEP_HELP=$H timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02bd_x400_h$H.log 2>&1
  echo "help=$H x400: $(grep -E "admm_bstep" $O/r02bd_x400_h$H.log)"
done
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py -q -x > $O/r02bd_tests.log 2>&1
tail -2 $O/r02bd_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c3_full or x400" > $O/r02bd_full.log 2>&1
tail -2 $O/r02bd_full.log
