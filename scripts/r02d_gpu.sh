#!/bin/bash
# round-2 pass d: warp-parallel Schur solve + p-update ILP (x400 heavy columns),
# PCG per-iteration kernel captures at C3, full GPU suite
set -x
O=gpurun_out
python -m pytest tests -q -m gpu -x > $O/r02d_gpu_tests.log 2>&1
EPC_BSTEP_TAIL=1 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 > $O/r02d_probe_x400.log 2>&1
python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02d_probe_x400_prod.log 2>&1
python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02d_probe_c3_prod.log 2>&1
EPC_PCG_LOOP=0 ncu --set full --clock-control none -k regex:"pcg_hvp|pcg_update_bj" --launch-skip 2 -c 2 -o $O/r02d_pcg_parts_c3 -f \
    python scripts/probe_gn.py --config C3 --ncu > $O/r02d_pcg_parts_ncu.log 2>&1
du -sh $O/*
