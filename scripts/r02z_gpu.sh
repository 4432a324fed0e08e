#!/bin/bash
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_update_ws -s 30 -c 1 \
  -o $O/r02z2_update_ws -f python scripts/probe_pcg.py C3 > $O/r02z2_ncu.log 2>&1
tail -2 $O/r02z2_ncu.log
