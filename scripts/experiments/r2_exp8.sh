#!/bin/bash
O=gpurun_out
N=1024 B=16 FFG_GROUP=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide1024b -f python scripts/profile_step.py > $O/ncu_w1024b.log 2>&1
