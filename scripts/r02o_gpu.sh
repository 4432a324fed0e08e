#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests -q -m gpu > $O/r02o_gpu_tests.log 2>&1
tail -5 $O/r02o_gpu_tests.log
