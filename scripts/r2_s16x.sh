#!/bin/bash
# 16-worker epilogue with X_l staged by cp.async during the MMAs: parity tests, A/B vs HEAD (base.so), timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_rowblock.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/s16x_tests.log
FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so timeout 120 python scripts/item_timeline.py 1024 > gpurun_out/tl1024_s16x.txt 2>&1
bash scripts/r2_ab.sh base "1024 1 MIXED_EMULATED" "256 1 MIXED_EMULATED" "2048 1 MIXED_EMULATED" "1024 4 MIXED_EMULATED" "1024 1 BF16" "512 64 MIXED_EMULATED" "1024 16 MIXED_EMULATED" > gpurun_out/s16x_ab.log 2>&1
