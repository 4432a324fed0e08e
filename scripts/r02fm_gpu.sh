#!/bin/bash
# C4 (64 pairs, one GPU) with and without the longest-columns-first order
set -x
O=gpurun_out
for ms in 1e9 5; do
EPC_LPT_MIN_MS=$ms python bench.py --config C4 --steps 3 --warmup 3 --no-gn --no-f32 --no-x400 --no-cpu-baseline > $O/r02fm_bench_c4_lpt$ms.json 2> $O/r02fm_bench_c4_lpt$ms.err
EPC_LPT_MIN_MS=$ms python bench.py --config C4 --scale 400 --iters 20 --steps 2 --warmup 3 --no-gn --no-f32 --no-x400 --no-cpu-baseline > $O/r02fm_bench_c4x400_lpt$ms.json 2> $O/r02fm_bench_c4x400_lpt$ms.err
done
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/r02fm_bench_c4*.json')):
    try:
        d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['config'].get('workload'))
    except Exception as e: print(f, 'ERR', e)
P
