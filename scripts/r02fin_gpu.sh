#!/bin/bash
# round-2 final pass: both arms at the driver's settings, launch list, PCG C3 parts capture
set -x
O=gpurun_out
P=${1:-r02fin}
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-gn-c3 --no-f32 --no-x400 --no-cpu-baseline > $O/${P}_launch_run.log 2>&1
ncu --set full --clock-control none -k regex:"pcg_hvp|pcg_update_ws" --launch-skip 2 -c 2 -o $O/${P}_pcg_parts_c3 -f \
    python scripts/probe_gn.py --config C3 --ncu > $O/${P}_pcg_parts_ncu.log 2>&1
ls -la $O | grep $P
