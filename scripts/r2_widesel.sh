#!/bin/bash
# wide vs pair (16-worker / 8+8-warp) kernels around the selection threshold
for r in 1 2; do
  for c in "2048 16 MIXED_EMULATED" "2048 1 BF16" "2048 16 BF16" "3072 1 MIXED_EMULATED" "4096 1 BF16" "4096 2 MIXED_EMULATED"; do
    echo "wide | $c | $(FFG_WIDE=1 timeout 120 python scripts/k2_time.py $c 4 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
    echo "s16 | $c | $(FFG_WIDE=0 FFG_S16=1 timeout 120 python scripts/k2_time.py $c 4 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
    echo "v0 | $c | $(FFG_WIDE=0 FFG_S16=0 timeout 120 python scripts/k2_time.py $c 4 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done 2>&1 | tee gpurun_out/widesel.log
