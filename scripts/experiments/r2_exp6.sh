#!/bin/bash
O=gpurun_out
FFG_GROUP=16 FFG_NORMAL_KSTEP=16 timeout 300 python scripts/wide_check.py 1024x16 512x128 4096x1 > $O/exp6.txt 2>&1
FFG_NORMAL_KSTEP=8 timeout 300 python scripts/wide_check.py 1024x16 >> $O/exp6.txt 2>&1
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
FFG_GROUP=16 MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 512x128 >> $O/exp6.txt 2>&1
