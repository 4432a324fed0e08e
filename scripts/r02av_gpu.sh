#!/bin/bash
# full GPU suite + smoke on the current tree
O=gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > $O/r02av_tests_gpu.log 2>&1
tail -4 $O/r02av_tests_gpu.log
timeout 600 python -c "import __graft_entry__ as e; e.smoke()" > $O/r02av_smoke.log 2>&1; echo "smoke rc=$?"
tail -3 $O/r02av_smoke.log
