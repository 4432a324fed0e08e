#!/bin/bash
# A/Bs: fused fwd2 with backoff, gated on the previous b-step length (default 12 ms) vs always vs off;
# DCT GEMM double-buffered K slabs (main build) vs single buffer (scripts/_var/nodb.so); then the GPU suite
set -x
O=gpurun_out
P=${1:-r02db}
mkdir -p $O
EPC_FUSE_FWD2=0 timeout 600 python scripts/ab_fuse_fwd2.py > $O/${P}_ab.log 2>&1
timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_ab.log 2>&1
EPC_FUSE_MAX_MS=1e9 timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_ab.log 2>&1
EPC_FUSE_FWD2=0 EPC_LIB=scripts/_var/nodb.so timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_ab.log 2>&1
cat $O/${P}_ab.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/${P}_gputests.log 2>&1
tail -3 $O/${P}_gputests.log
