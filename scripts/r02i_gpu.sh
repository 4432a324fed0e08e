#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests/test_gpu_admm.py tests/test_gpu_golden.py -q -x > $O/r02i_tests.log 2>&1
python scripts/probe_qp.py > $O/r02i_qp.log 2>&1
python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02i_probe_x400_prod.log 2>&1
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02i_probe_c3_prod.log 2>&1
EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 > $O/r02i_probe_x400.log 2>&1
python -m pytest tests/test_gpu_fullsize.py -q -x -k "x400 or batch" > $O/r02i_fullsize.log 2>&1
EPC_PCG_LOOP=0 EPC_PCG_SEG=0 python scripts/probe_gn.py --config C3 > $O/r02i_gn_c3_noseg.log 2>&1
python scripts/probe_gn.py --config C3 > $O/r02i_gn_c3.log 2>&1
grep -h "unprofiled" $O/r02i_gn_*.log
