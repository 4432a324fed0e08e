#!/bin/bash
set -x
O=gpurun_out
python -m pytest tests/test_gpu_admm.py -q -x > $O/r02m_tests.log 2>&1
for i in 1 2; do
for V in now r1 ser0 ser32; do
  if [ $V = now ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02m_c3_${V}_$i.log 2>&1
done
done
for V in now ser0 ser32; do
  if [ $V = now ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L python scripts/probe_admm.py --config C3 --scale 400 --iters 100 --prod > $O/r02m_x400_${V}.log 2>&1
done
python scripts/probe_qp.py > $O/r02m_qp.log 2>&1
for f in $O/r02m_c3_*.log $O/r02m_x400_*.log; do echo "$f $(grep admm_bstep $f)"; done
