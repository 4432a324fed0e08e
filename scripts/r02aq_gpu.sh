#!/bin/bash
O=gpurun_out
timeout 600 python scripts/probe_ls.py C3 1.0 100 > $O/r02aq_ls_c3.log 2>&1
timeout 600 python scripts/probe_ls.py C3 400.0 30 > $O/r02aq_ls_x400.log 2>&1
cat $O/r02aq_ls_c3.log $O/r02aq_ls_x400.log
