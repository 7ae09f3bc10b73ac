#!/bin/bash
O=gpurun_out
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
: > $O/exp13.txt
for d in 0 512 736 1; do
  echo "dbg=$d" >> $O/exp13.txt
  FFG_DEBUG_K2=$d MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp13.txt 2>&1
done
