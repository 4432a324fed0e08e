#!/bin/bash
# round-2 measurement pass b: bench (both arms), GN-PCG loop captures, launch list
set -x
O=gpurun_out
python bench.py --steps 20 --warmup 5 > $O/r02b_bench.json 2> $O/r02b_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/r02b_bench_ref.json 2> $O/r02b_bench_ref.err
for C in C2 C3; do
  python scripts/probe_gn.py --config $C --ncu > $O/r02b_pcg_${C}_iters.txt 2>&1
  ncu --set full --clock-control none --import-source on -k regex:pcg_loop -c 1 -o $O/r02b_pcg_$C -f \
      python scripts/probe_gn.py --config $C --ncu > $O/r02b_pcg_${C}_ncu.log 2>&1
done
python scripts/probe_gn.py --config C3 > $O/r02b_gn_c3_probe.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/r02b_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-f32 --no-x400 --no-cpu-baseline > $O/r02b_launch_run.log 2>&1
ls -la $O
