#!/bin/bash
# tail help v2 (bitmap discovery, hoisted queue check): A/B vs the HEAD build, bitwise tests
O=gpurun_out
mkdir -p $O
run() {  # name env...
  local n=$1; shift
  env "$@" timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02be_c3_$n.log 2>&1
  echo "$n C3: $(grep -E "^admm|admm_bstep" $O/r02be_c3_$n.log | tr '\n' ' ')"
}
runx() {
  local n=$1; shift
  env "$@" timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02be_x400_$n.log 2>&1
  echo "$n x400: $(grep -E "admm_bstep" $O/r02be_x400_$n.log)"
}
run base EPC_LIB=scripts/_var/base.so
run h1 EPC_BSTEP_HELP=1
run h0 EPC_BSTEP_HELP=0
run base EPC_LIB=scripts/_var/base.so
run h1 EPC_BSTEP_HELP=1
runx base EPC_LIB=scripts/_var/base.so
runx h1 EPC_BSTEP_HELP=1
runx h0 EPC_BSTEP_HELP=0
timeout 1200 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_admm_loop.py -q -x > $O/r02be_tests.log 2>&1
tail -2 $O/r02be_tests.log
