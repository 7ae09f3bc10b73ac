#!/bin/bash
# config 4 (512 x N=512): K2 time vs L2-resident group size, pair (default) and wide kernels
mkdir -p gpurun_out
for mode in MIXED_EMULATED BF16; do
  for g in 6 10 15 20 30 43 64; do
    echo "pair G=$g $(FFG_GROUP=$g timeout 120 python scripts/k2_time.py 512 512 $mode 5)"
  done
  for g in 8 16 32 64; do
    echo "wide G=$g $(FFG_WIDE=1 FFG_GROUP=$g timeout 120 python scripts/k2_time.py 512 512 $mode 5)"
  done
done 2>&1 | tee gpurun_out/cfg4_sweep.log
