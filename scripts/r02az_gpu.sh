#!/bin/bash
O=gpurun_out
timeout 900 python scripts/probe_admm.py --config C3 --scale 400 --iters 30 > $O/r02az_x400_phases.log 2>&1
head -4 $O/r02az_x400_phases.log
