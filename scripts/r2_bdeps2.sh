#!/bin/bash
# alternate block-granular dependencies off/on to separate the effect from clock drift
mkdir -p gpurun_out
for r in 1 2; do for bd in 0 1; do
  echo "== bd=$bd rep=$r"; FFG_BLOCKDEPS=$bd MODES=BF16,MIXED_EMULATED timeout 600 python scripts/wide_check.py 4096x1 8192x1 2>&1
  nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv,noheader
done; done | tee gpurun_out/bdeps_alt.log
