#!/bin/bash
# K2 memory-traffic sensitivity (measurement only)
c=${1:-1024x16}
for d in 0 64 128 192 224 240 16 32; do
  FFG_LIB_PATH=paper_2605_08523_b200/lib/var/lib_cur.so FFG_DEBUG_K2=$d timeout 100 python scripts/k2_variants.py $c 2>&1 | grep MIXED | sed "s/^.*\] //" | sed "s/^/dbg=$d /"
done
