#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_admm_loop.py tests/test_gpu_admm.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py -q -x -k "not c3_full and not x400" > $O/r02aj_tests.log 2>&1
tail -3 $O/r02aj_tests.log
