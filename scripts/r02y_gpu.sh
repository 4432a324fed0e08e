#!/bin/bash
# PCG update: warp-specialised pipelined kernel vs the single-role kernel
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gn.py -q -x > $O/r02y2_tests_gn.log 2>&1
tail -3 $O/r02y2_tests_gn.log
for i in 1 2; do
for W in 1 0; do
  EPC_PCG_WS=$W timeout 300 python scripts/probe_pcg.py C3 > $O/r02y2_pcg_ws${W}_$i.log 2>&1
  echo "ws=$W $i: $(grep block $O/r02y2_pcg_ws${W}_$i.log)"
done
done
for W in 1 0; do
  for C in C2 C3; do
    EPC_PCG_WS=$W timeout 300 python scripts/probe_gn.py --config $C > $O/r02y2_gn_ws${W}_$C.log 2>&1
    echo "ws=$W $C: $(grep -E "^GN|pcg_update|pcg_loop" $O/r02y2_gn_ws${W}_$C.log | tr "\n" " ")"
  done
done
