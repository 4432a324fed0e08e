#!/bin/bash
# PCG bandwidth variants (per-iteration kernels and the persistent loop) at C3
set -x
O=gpurun_out
for V in default hvpU1 hvpU4 hvpU4m3; do
  if [ $V = default ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L python scripts/probe_gn.py --config C3 > $O/r02f_gn_$V.log 2>&1
  env $L EPC_PCG_LOOP=0 python scripts/probe_gn.py --config C3 > $O/r02f_gn_${V}_noloop.log 2>&1
done
python -m pytest tests/test_gpu_gn.py -q > $O/r02f_gn_tests.log 2>&1
grep -h "unprofiled\|pcg_loop \|pcg_hvp \|pcg_update " $O/r02f_gn_*.log
python scripts/probe_qp.py > $O/r02f_qp.log 2>&1
EPC_LIB=scripts/_var/noschur.so python scripts/probe_qp.py > $O/r02f_qp_noschur.log 2>&1
