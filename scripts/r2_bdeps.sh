#!/bin/bash
# wide kernel block-granular dependencies: on/off at single-matrix N=2048/4096/8192, then the wide GPU tests
set -x
mkdir -p gpurun_out
for bd in 0 1; do
  FFG_BLOCKDEPS=$bd timeout 600 python scripts/wide_check.py 2048x1 4096x1 8192x1 2>&1 | tee gpurun_out/bdeps_$bd.log
done
FFG_BLOCKDEPS=1 timeout 300 python scripts/wide_check.py 4096x2 2048x4 2>&1 | tee gpurun_out/bdeps_batch.log
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/bdeps_tests.log
