#!/bin/bash
# drain/worker chunk waits: spin (default build) vs suspend-hint try_wait (FFG_DRAIN_SLEEP=1 variant)
mkdir -p gpurun_out
FFG_LIB_PATH=paper_2605_08523_b200/lib/var/profsl.so timeout 120 python scripts/item_timeline.py 1024 > gpurun_out/tl1024_sleep.txt 2>&1
for r in 1 2; do for lib in default sl; do
  L=""; [ $lib = sl ] && L=paper_2605_08523_b200/lib/var/sl.so
  for c in "1024 1" "1024 16" "256 1" "4096 1" "2048 1" "512 512"; do
    echo "$lib $c $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py $c MIXED_EMULATED 10)"
  done
  echo "$lib 1024 16 BF16 $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py 1024 16 BF16 10)"
  echo "$lib 4096 1 BF16 $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py 4096 1 BF16 10)"
done; done 2>&1 | sed 's/"lib": "[^"]*", //' | tee gpurun_out/sleep.log
