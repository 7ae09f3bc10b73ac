#!/bin/bash
O=gpurun_out
export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so
: > $O/exp11.txt
for d in 0 128 64 32 224; do
  echo "dbg=$d" >> $O/exp11.txt
  FFG_DEBUG_K2=$d timeout 300 python scripts/wide_roles.py 1024x16 >> $O/exp11.txt 2>&1
done
