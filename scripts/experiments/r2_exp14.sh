#!/bin/bash
O=gpurun_out
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
: > $O/exp14.txt
for d in 0 736; do
  echo "dbg=$d" >> $O/exp14.txt
  FFG_DEBUG_K2=$d MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp14.txt 2>&1
done
