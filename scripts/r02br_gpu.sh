#!/bin/bash
# late b-step captures of the current build (source-level: hot/cold code map)
O=gpurun_out
P=${1:-r02br}
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 90 -c 1 -o $O/${P}_bstep_c3_late -f \
    python scripts/probe_admm.py --config C3 --iters 91 --prod > $O/${P}_bstep_c3_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:admm_bstep --launch-skip 60 -c 1 -o $O/${P}_bstep_x400_late -f \
    python scripts/probe_admm.py --config C3 --scale 400 --iters 61 --prod > $O/${P}_bstep_x400_ncu.log 2>&1
ls -la $O | grep $P
