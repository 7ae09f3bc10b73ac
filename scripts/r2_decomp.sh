#!/bin/bash
# bench-config K2 time with epilogue memory streams removed (FFG_DEBUG_K2 measurement bits; results invalid):
# 32 = no hi/lo TMA stores, 64 = no A reductions, 128 = no X_l loads
mkdir -p gpurun_out
for r in 1 2; do for d in 0 32 64 128 224; do
  echo "dbg=$d $(FFG_DEBUG_K2=$d timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 20)"
done; done 2>&1 | sed 's/"lib": "default", //' | tee gpurun_out/decomp.log
