#!/bin/bash
O=gpurun_out
timeout 900 python scripts/probe_chained.py 1.0 30 > $O/r02as_chained.log 2>&1
cat $O/r02as_chained.log
