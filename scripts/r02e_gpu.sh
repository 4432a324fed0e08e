#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests -q -m gpu > $O/r02e_gpu_tests.log 2>&1
EPC_F32_ACC64=1 python -m pytest tests/test_gpu_admm_f32.py -q -s > $O/r02e_f32_acc64.log 2>&1
EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 > $O/r02e_probe_x400.log 2>&1
python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02e_probe_x400_prod.log 2>&1
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02e_probe_c3_prod.log 2>&1
python scripts/probe_f32.py C3 100 > $O/r02e_probe_f32.log 2>&1
EPC_F32_ACC64=1 python scripts/probe_f32.py C3 100 > $O/r02e_probe_f32_acc64.log 2>&1
