#!/bin/bash
# round-2 bench pass: both arms at the driver's settings, launch list, b-step captures
set -x
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r02n_bench.json 2> $O/r02n_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/r02n_bench_ref.json 2> $O/r02n_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02n_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-f32 --no-x400 --no-cpu-baseline > $O/r02n_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 90 -c 1 -o $O/r02n_bstep_c3_late -f \
    python scripts/probe_admm.py --config C3 --iters 91 --prod > $O/r02n_bstep_c3_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 60 -c 1 -o $O/r02n_bstep_x400_late -f \
    python scripts/probe_admm.py --config C3 --scale 400 --iters 61 --prod > $O/r02n_bstep_x400_ncu.log 2>&1
ls -la $O | grep r02n
