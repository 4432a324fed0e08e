#!/bin/bash
# ncu source-level capture of the C3 PCG update kernel (probe_pcg exited 0 in r02s)
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_update_bj -s 30 -c 1 \
  -o $O/r02t_update python scripts/probe_pcg.py C3 > $O/r02t_ncu.log 2>&1
tail -3 $O/r02t_ncu.log
EPC_LIB=scripts/_var/pcgnomem.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_update_bj -s 30 -c 1 \
  -o $O/r02t_update_nomem python scripts/probe_pcg.py C3 > $O/r02t_ncu_nomem.log 2>&1
tail -3 $O/r02t_ncu_nomem.log
ls -la $O/*.ncu-rep
