#!/bin/bash
O=gpurun_out
N=1024 B=16 FFG_DEBUG_K2=736 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide_nomem -f python scripts/profile_step.py > $O/ncu_nomem.log 2>&1
N=1024 B=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide1024c -f python scripts/profile_step.py > $O/ncu_w1024c.log 2>&1
