#!/bin/bash
# closing pass with the longest-columns-first order on (default EPC_LPT_MIN_MS=5):
# GPU suite + smoke, bench, launch list, late x400 capture
set -x
O=gpurun_out
P=${1:-r02fk}
mkdir -p $O profiles
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${P}_smoke.log 2>&1
tail -2 $O/${P}_smoke.log
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-gn-c3 --no-f32 --no-x400 --no-cpu-baseline > $O/${P}_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 60 -c 1 -o $O/${P}_bstep_x400_late -f \
    python scripts/probe_admm.py --config C3 --scale 400 --iters 61 --prod > $O/${P}_bstep_x400_ncu.log 2>&1
python scripts/probe_iter_profile.py --scale 400 > $O/${P}_iter_profile_x400.log 2>&1
ls -la $O | grep $P
