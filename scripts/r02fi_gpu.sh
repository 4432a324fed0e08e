#!/bin/bash
# longest-columns-first order in the bulk-bound launches (EPC_LPT_MIN_MS): A/B with bitwise digests
set -x
O=gpurun_out
P=${1:-r02fi}
mkdir -p $O
: > $O/${P}_lpt_ab.log
for ms in 1e9 0 3 5 8; do
  echo "== EPC_LPT_MIN_MS=$ms" >> $O/${P}_lpt_ab.log
  EPC_LPT_MIN_MS=$ms timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_lpt_ab.log 2>&1
done
grep "==\|median" $O/${P}_lpt_ab.log
EPC_LPT_MIN_MS=5 EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --iters 16 --prod 2>&1 | grep "bstep tail" > $O/${P}_tail_it16.log
cat $O/${P}_tail_it16.log
