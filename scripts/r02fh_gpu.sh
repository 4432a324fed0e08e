#!/bin/bash
# early-trajectory b-step (iterations 1-16 of C3: 9-12 ms launches, 45% of the
# b-step's time in the first 25 iterations): phase split and ncu captures
set -x
O=gpurun_out
python scripts/probe_admm.py --config C3 --iters 16 > $O/r02fh_phases_it16.log 2>&1
python scripts/probe_admm.py --config C3 --iters 100 > $O/r02fh_phases_it100.log 2>&1
for skip in 9 15; do
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip $skip -c 1 -o $O/r02fh_bstep_c3_it$((skip-1)) -f \
    python scripts/probe_admm.py --config C3 --iters $((skip-1)) --prod > $O/r02fh_ncu_$skip.log 2>&1
python scripts/summarize_ncu.py capture $O/r02fh_bstep_c3_it$((skip-1)).ncu-rep $O/r02fh_bstep_c3_it$((skip-1))_ncu.json
done
EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --iters 16 --prod > $O/r02fh_tail_it16.log 2>&1
tail -5 $O/r02fh_phases_it16.log
