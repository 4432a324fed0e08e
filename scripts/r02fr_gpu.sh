#!/bin/bash
# same-box A/B: library at 5150dab (prev), HEAD, HEAD without the critical-column code (-DEPC_NO_CRIT)
set -x
O=gpurun_out
: > $O/r02fr_ab.log
for rep in 1 2; do
  for lib in paper_1607_00531_b200/libepicorr_b200_prev.so scripts/_var/nocrit.so paper_1607_00531_b200/libepicorr_b200.so; do
    EPC_LIB=$PWD/$lib timeout 600 python scripts/ab_fuse_fwd2.py 2>&1 | grep median | sed "s#lib=[^ ]*/#lib=#" >> $O/r02fr_ab.log
  done
done
cat $O/r02fr_ab.log
