#!/bin/bash
O=gpurun_out
N=512 B=128 timeout 600 ncu --set full --clock-control none -k regex:mlsp2_pair -s 1 -c 1 -o $O/pair512 -f python scripts/profile_step.py > $O/ncu_p512.log 2>&1
for g in 8 16 24 32 48; do FFG_GROUP=$g timeout 120 python scripts/k2_time.py 512 128 MIXED_EMULATED 5; done > $O/exp19_g.txt 2>&1
for g in 8 16 24 32 48; do FFG_GROUP=$g timeout 120 python scripts/k2_time.py 512 128 BF16 5; done >> $O/exp19_g.txt 2>&1
