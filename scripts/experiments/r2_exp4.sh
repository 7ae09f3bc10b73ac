#!/bin/bash
O=gpurun_out
N=512 B=64 FFG_WIDE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide512 -f python scripts/profile_step.py > $O/ncu_w512.log 2>&1
N=1024 B=16 FFG_GROUP=16 FFG_WIDE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide1024 -f python scripts/profile_step.py > $O/ncu_w1024.log 2>&1
