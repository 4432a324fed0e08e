#!/bin/bash
# round-2 pass c: per-column b-step records for the scheduling study, fp32 GEMM check
set -x
O=gpurun_out
D=/tmp/r02c
mkdir -p $D
export EPC_BSTEP_DUMP_EVERY=10
EPC_BSTEP_TAIL=1 EPC_BSTEP_DUMP=$D/dump_c3.bin python scripts/probe_admm.py --config C3 --iters 100 > $O/r02c_probe_c3.log 2>&1
EPC_BSTEP_TAIL=1 EPC_BSTEP_DUMP=$D/dump_x400.bin python scripts/probe_admm.py --config C3 --scale 400 --iters 60 > $O/r02c_probe_x400.log 2>&1
python scripts/analyze_bstep_dump.py $D/dump_c3.bin > $O/r02c_sched_c3.log 2>&1
python scripts/analyze_bstep_dump.py $D/dump_x400.bin > $O/r02c_sched_x400.log 2>&1
gzip -c $D/dump_c3.bin > $O/r02c_dump_c3.bin.gz
gzip -c $D/dump_x400.bin > $O/r02c_dump_x400.bin.gz
python -m pytest tests/test_gpu_admm_f32.py tests/test_gpu_gn.py -q -s > $O/r02c_f32_gn_tests.log 2>&1
python bench.py --steps 5 --warmup 2 --no-x400 --no-cpu-baseline > $O/r02c_bench.json 2> $O/r02c_bench.err
python scripts/probe_gn.py --config C3 > $O/r02c_gn_c3_probe.log 2>&1
EPC_PCG_SEG=0 python scripts/probe_gn.py --config C3 > $O/r02c_gn_c3_probe_noseg.log 2>&1
du -sh $O/*
