#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests/test_gpu_gn.py tests/test_gpu_admm_f32.py -q > $O/r02g_tests.log 2>&1
python scripts/probe_gn.py --config C3 > $O/r02g_gn_c3.log 2>&1
python scripts/probe_gn.py --config C2 > $O/r02g_gn_c2.log 2>&1
python scripts/probe_qp.py > $O/r02g_qp.log 2>&1
EPC_LIB=scripts/_var/noschur.so python scripts/probe_qp.py > $O/r02g_qp_noschur.log 2>&1
ncu --set full --clock-control none -k regex:"pcg_hvp|pcg_update_bj" --launch-skip 2 -c 2 -o $O/r02g_pcg_parts_c3 -f \
    python scripts/probe_gn.py --config C3 --ncu > $O/r02g_pcg_parts_ncu.log 2>&1
