#!/bin/bash
O=gpurun_out
FFG_WIDE=0 timeout 300 python scripts/wide_check.py 1024x16 512x128 256x1 1024x1 > $O/exp23.txt 2>&1
N=1024 B=16 timeout 600 ncu --metrics sass__inst_executed_local_loads,sass__inst_executed_local_stores,gpu__time_duration.sum,lts__t_sectors.sum -k regex:mlsp2_pair -s 1 -c 1 --csv python scripts/profile_step.py > $O/exp23_ncu.csv 2>/dev/null
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > $O/b23.json 2>/dev/null
