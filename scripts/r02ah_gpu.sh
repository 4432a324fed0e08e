#!/bin/bash
# pipelined ADMM loop: bitwise tests, then timing vs the synchronous loop
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_admm_loop.py tests/test_gpu_admm.py tests/test_gpu_golden.py -q -x > $O/r02ah_tests.log 2>&1
tail -3 $O/r02ah_tests.log
timeout 900 python scripts/probe_loop.py > $O/r02ah_loop.log 2>&1
cat $O/r02ah_loop.log
