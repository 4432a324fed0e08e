#!/bin/bash
# fused forward axis-2 transform in the b-step's drain: A/B (time + bitwise digests), then the GPU suite
set -x
O=gpurun_out
P=${1:-r02fu}
mkdir -p $O
EPC_FUSE_FWD2=0 timeout 600 python scripts/ab_fuse_fwd2.py > $O/${P}_ab.log 2>&1
EPC_FUSE_FWD2=1 timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_ab.log 2>&1
cat $O/${P}_ab.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
