#!/bin/bash
# critical-column SM reservation A/B (bitwise digests must agree across modes)
set -x
O=gpurun_out
: > $O/r02fo_crit_ab.log
for c in 0 1.0 0.8 1.3; do
  EPC_LPT_CRIT=$c timeout 600 python scripts/ab_lpt_crit.py >> $O/r02fo_crit_ab.log 2>&1
done
cat $O/r02fo_crit_ab.log
EPC_BSTEP_TAIL=1 timeout 300 python scripts/probe_admm.py --config C3 --scale 400 --iters 40 --prod 2>&1 | grep -A1 "bstep tail" | tail -6 > $O/r02fo_tail_x400.log
cat $O/r02fo_tail_x400.log
