#!/bin/bash
O=gpurun_out
FFG_WIDE=1 timeout 300 python scripts/wide_check.py 1024x16 1024x1 512x128 4096x1 > $O/exp16.txt 2>&1
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
FFG_WIDE=1 MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp16.txt 2>&1
