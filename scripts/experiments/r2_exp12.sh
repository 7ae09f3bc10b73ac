#!/bin/bash
O=gpurun_out
timeout 300 python scripts/wide_check.py 1024x16 2048x4 4096x1 > $O/exp12.txt 2>&1
FFG_NORMAL_KSTEP=16 MODES=MIXED_EMULATED timeout 300 python scripts/wide_check.py 1024x16 >> $O/exp12.txt 2>&1
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp12.txt 2>&1
