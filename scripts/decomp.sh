#!/bin/bash
# K2 time decomposition (measurement only; dbg variants give wrong results by design).
# usage: bash scripts/decomp.sh CASE lib...
c=$1; shift
for L in "$@"; do
  export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/$L
  for d in 0 1 4 32 64 96 97 16 17; do
    FFG_DEBUG_K2=$d timeout 100 python scripts/k2_variants.py $c 2>&1 | grep -E "MIXED" | sed "s/^/$L dbg=$d /" | sed 's/\[.*\]//'
  done
  FFG_EXACT_DRAIN_LAYERS=0 timeout 100 python scripts/k2_variants.py $c 2>&1 | grep -E "MIXED" | sed "s/^/$L exact=0 /" | sed 's/\[.*\]//'
done
