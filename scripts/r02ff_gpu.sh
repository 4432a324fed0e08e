#!/bin/bash
# round-2 closing pass (fused forward axis-2 DCT, double-buffered dual GEMM):
# late b-step capture first (the bench's roofline reads its summary), GPU suite + smoke,
# both bench arms, launch list, late x400 capture
set -x
O=gpurun_out
P=${1:-r02ff}
mkdir -p $O profiles
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 90 -c 1 -o $O/${P}_bstep_c3_late -f \
    python scripts/probe_admm.py --config C3 --iters 91 --prod > $O/${P}_bstep_c3_ncu.log 2>&1
python scripts/summarize_ncu.py capture $O/${P}_bstep_c3_late.ncu-rep profiles/${P}_bstep_c3_late_ncu.json
cp profiles/${P}_bstep_c3_late_ncu.json $O/
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${P}_smoke.log 2>&1
tail -2 $O/${P}_smoke.log
python bench.py --steps 20 --warmup 5 > $O/${P}_bench.json 2> $O/${P}_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${P}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-gn --no-gn-c3 --no-f32 --no-x400 --no-cpu-baseline > $O/${P}_launch_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 60 -c 1 -o $O/${P}_bstep_x400_late -f \
    python scripts/probe_admm.py --config C3 --scale 400 --iters 61 --prod > $O/${P}_bstep_x400_ncu.log 2>&1
ls -la $O | grep $P
