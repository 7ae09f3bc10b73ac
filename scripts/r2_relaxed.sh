#!/bin/bash
# relaxed dependency polls + one acquire fence: K2 times on the single-matrix / small configs, timeline, wide tests
mkdir -p gpurun_out
FFG_LIB_PATH=paper_2605_08523_b200/lib/var/prof.so timeout 120 python scripts/item_timeline.py 1024 > gpurun_out/tl1024_relaxed.txt 2>&1
for c in "1024 1" "256 1" "2048 1" "4096 1" "1024 16" "512 512"; do
  echo "$c $(timeout 120 python scripts/k2_time.py $c MIXED_EMULATED 10)"
done 2>&1 | sed 's/"lib": "[^"]*", //' | tee gpurun_out/relaxed.log
echo "4096 1 BF16 $(timeout 120 python scripts/k2_time.py 4096 1 BF16 10)" | tee -a gpurun_out/relaxed.log
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3 | tee -a gpurun_out/relaxed.log
