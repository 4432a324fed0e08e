#!/bin/bash
# A/B: the RM=4 non-dual DCT GEMMs at three resident CTAs per SM (scripts/_var/minb3.so) vs two; batch tests
set -x
O=gpurun_out
P=${1:-r02mb}
mkdir -p $O
timeout 600 python scripts/ab_fuse_fwd2.py > $O/${P}_ab.log 2>&1
EPC_LIB=scripts/_var/minb3.so timeout 600 python scripts/ab_fuse_fwd2.py >> $O/${P}_ab.log 2>&1
cat $O/${P}_ab.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k batch > $O/${P}_tests.log 2>&1
tail -3 $O/${P}_tests.log
