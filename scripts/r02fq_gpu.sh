#!/bin/bash
# same-box A/B of the round's last three changes against the library built at 5150dab (before them):
# paper_1607_00531_b200/libepicorr_b200_prev.so through EPC_LIB; interleaved twice
set -x
O=gpurun_out
: > $O/r02fq_prev_ab.log
for rep in 1 2; do
  EPC_LIB=$PWD/paper_1607_00531_b200/libepicorr_b200_prev.so timeout 600 python scripts/ab_fuse_fwd2.py 2>&1 | grep median >> $O/r02fq_prev_ab.log
  timeout 600 python scripts/ab_fuse_fwd2.py 2>&1 | grep median >> $O/r02fq_prev_ab.log
done
cat $O/r02fq_prev_ab.log
