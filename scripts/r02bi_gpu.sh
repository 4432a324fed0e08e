#!/bin/bash
# tail help stats (dev aid EPC_HELP_STATS)
O=gpurun_out
mkdir -p $O
EPC_HELP_STATS=1 timeout 300 python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02bi_c3.log 2>&1
grep -E "help stats|admm_bstep" $O/r02bi_c3.log | tail -4
EPC_HELP_STATS=1 timeout 600 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 --prod > $O/r02bi_x400.log 2>&1
grep -E "help stats|admm_bstep" $O/r02bi_x400.log | tail -3
