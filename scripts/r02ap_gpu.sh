#!/bin/bash
O=gpurun_out
timeout 600 python scripts/probe_admm.py --config C3 --iters 100 > $O/r02ap_c3_phases.log 2>&1
head -8 $O/r02ap_c3_phases.log
