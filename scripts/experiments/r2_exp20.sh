#!/bin/bash
O=gpurun_out
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
: > $O/exp20.txt
for d in 0 2 16 18 738; do
  echo "dbg=$d" >> $O/exp20.txt
  FFG_WIDE=1 FFG_DEBUG_K2=$d MODES=MIXED_EMULATED timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp20.txt 2>&1
done
