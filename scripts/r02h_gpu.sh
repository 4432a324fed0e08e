#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests/test_gpu_multi_abi.py tests/test_gpu_gn.py tests/test_gpu_admm_f32.py tests/test_gpu_admm.py -q > $O/r02h_tests.log 2>&1
python scripts/probe_qp.py > $O/r02h_qp.log 2>&1
EPC_LIB=scripts/_var/noschur.so python scripts/probe_qp.py > $O/r02h_qp_noschur.log 2>&1
python scripts/probe_gn.py --config C2 > $O/r02h_gn_c2.log 2>&1
EPC_PCG_SEG=0 python scripts/probe_gn.py --config C2 > $O/r02h_gn_c2_noseg.log 2>&1
EPC_LIB=scripts/_var/hvpbatchloop.so python scripts/probe_gn.py --config C2 > $O/r02h_gn_c2_batchloop.log 2>&1
python scripts/probe_gn.py --config C3 > $O/r02h_gn_c3.log 2>&1
grep -h "unprofiled" $O/r02h_gn_*.log
