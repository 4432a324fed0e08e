#!/bin/bash
set -x
O=gpurun_out
python scripts/probe_gn.py --config C3 > $O/r02j_gn_c3.log 2>&1
python scripts/probe_gn.py --config C2 > $O/r02j_gn_c2.log 2>&1
EPC_PCG_SEG=0 python scripts/probe_gn.py --config C2 > $O/r02j_gn_c2_noseg.log 2>&1
EPC_PCG_BAL=0 python scripts/probe_gn.py --config C2 > $O/r02j_gn_c2_nobal.log 2>&1
EPC_PCG_BAL=0 EPC_PCG_SEG=0 python scripts/probe_gn.py --config C2 > $O/r02j_gn_c2_nobal_noseg.log 2>&1
python -m pytest tests/test_gpu_gn.py -q > $O/r02j_gn_tests.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize_smoke.py > $O/r02j_sanitizer_$t.log 2>&1
  echo "$t rc=$?" >> $O/r02j_sanitizer_rc.txt
done
grep -h "unprofiled" $O/r02j_gn_*.log
