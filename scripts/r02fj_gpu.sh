#!/bin/bash
# LPT order keyed on the larger of the last two launches' costs: A/B with bitwise digests
set -x
O=gpurun_out
P=${1:-r02fj}
mkdir -p $O
: > $O/${P}_lpt_ab.log
for cfg in "5 0" "5 1" "3 1" "0 1"; do
  set -- $cfg
  echo "== EPC_LPT_MIN_MS=$1 EPC_LPT_TWO=$2" >> $O/${P}_lpt_ab.log
  EPC_LPT_MIN_MS=$1 EPC_LPT_TWO=$2 timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_lpt_ab.log 2>&1
done
grep "==\|median" $O/${P}_lpt_ab.log
EPC_LPT_MIN_MS=5 EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --iters 16 --prod 2>&1 | grep "bstep tail" > $O/${P}_tail_it16.log
tail -8 $O/${P}_tail_it16.log
EPC_LPT_MIN_MS=0 EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --iters 90 --prod 2>&1 | grep "bstep tail" | tail -6 > $O/${P}_tail_it90.log
cat $O/${P}_tail_it90.log
