#!/bin/bash
O=gpurun_out
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
FFG_GROUP=16 MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 > $O/exp5.txt 2>&1
MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 512x128 4096x1 256x1 >> $O/exp5.txt 2>&1
