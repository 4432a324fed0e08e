#!/bin/bash
# DCT GEMM: 8x8 register tiles per transform (EPC_GEMM_RN8 bit mask) - bitwise + timing
O=gpurun_out
EPC_GEMM_RN8=15 timeout 900 python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py -q -x > $O/r02ak_tests.log 2>&1
tail -2 $O/r02ak_tests.log
for R in 0 15; do
  EPC_GEMM_RN8=$R timeout 300 python scripts/probe_admm.py --config C3 --iters 20 --prod > $O/r02ak_c3_rn$R.log 2>&1
  echo "RN8=$R"; grep -E "dct_" $O/r02ak_c3_rn$R.log
done
