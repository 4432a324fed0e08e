#!/bin/bash
# closing pass with the critical-column reservation (EPC_LPT_CRIT default 0.8): A/B, GPU suite + smoke, bench
set -x
O=gpurun_out
P=${1:-r02fp}
: > $O/${P}_crit_ab.log
for c in 0 0.8; do
  EPC_LPT_CRIT=$c timeout 600 python scripts/ab_lpt_crit.py >> $O/${P}_crit_ab.log 2>&1
done
cat $O/${P}_crit_ab.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${P}_smoke.log 2>&1
tail -2 $O/${P}_smoke.log
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 60 -c 1 -o $O/${P}_bstep_x400_late -f \
    python scripts/probe_admm.py --config C3 --scale 400 --iters 61 --prod > $O/${P}_bstep_x400_ncu.log 2>&1
