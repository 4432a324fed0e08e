#!/bin/bash
# round-2 closing pass (longest-columns-first order on, critical-column reservation compiled out):
# GPU suite + smoke, both bench arms, launch list
set -x
O=gpurun_out
P=${1:-r02fs}
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${P}_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-gn-c3 --no-f32 --no-x400 --no-cpu-baseline > $O/${P}_launch_run.log 2>&1
