#!/bin/bash
# pair kernel: block-granular dependencies in multi-matrix groups (bench config, config 4), alternating
mkdir -p gpurun_out
for r in 1 2; do for bd in 0 1; do
  echo "bd=$bd 1024x16 $(FFG_BLOCKDEPS=$bd timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 20)"
  echo "bd=$bd 1024x16 G=16 $(FFG_GROUP=16 FFG_BLOCKDEPS=$bd timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 20)"
  echo "bd=$bd 512x512 $(FFG_BLOCKDEPS=$bd timeout 120 python scripts/k2_time.py 512 512 MIXED_EMULATED 5)"
  echo "bd=$bd 512x512 BF16 $(FFG_BLOCKDEPS=$bd timeout 120 python scripts/k2_time.py 512 512 BF16 5)"
done; done 2>&1 | tee gpurun_out/bd_pair.log
