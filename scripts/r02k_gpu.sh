#!/bin/bash
set -x
O=gpurun_out
EPC_GUARD=1 EPC_LIB=scripts/_var/canary.so python scripts/sanitize_smoke.py > $O/r02k_guard_canary.log 2>&1
echo "rc=$?" >> $O/r02k_guard_canary.log
EPC_GUARD=1 python scripts/sanitize_smoke.py > $O/r02k_guard_prod.log 2>&1
echo "rc=$?" >> $O/r02k_guard_prod.log
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02k_c3_now.log 2>&1
EPC_LIB=scripts/_var/r1.so python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02k_c3_r1.log 2>&1
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02k_c3_now2.log 2>&1
python scripts/probe_gn.py --config C2 > $O/r02k_gn_c2.log 2>&1
EPC_LIB=scripts/_var/r1.so python scripts/probe_gn.py --config C2 > $O/r02k_gn_c2_r1.log 2>&1
python scripts/probe_gn.py --config C3 > $O/r02k_gn_c3.log 2>&1
EPC_PCG_LOOP=0 ncu --set full --clock-control none -k regex:"pcg_hvp|pcg_update_bj" --launch-skip 2 -c 2 -o $O/r02k_pcg_parts_c3 -f \
    python scripts/probe_gn.py --config C3 --ncu > $O/r02k_pcg_parts_ncu.log 2>&1
grep -h "admm 100\|admm_bstep\|unprofiled" $O/r02k_*.log
