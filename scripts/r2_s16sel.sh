#!/bin/bash
# 16-worker (S16) vs 8+8-warp (V0) pair kernel after the control-warp register change: which wins where
for r in 1 2; do for s in 0 1; do
  for c in "1024 64 MIXED_EMULATED" "1536 4 MIXED_EMULATED" "1536 1 MIXED_EMULATED" "1024 16 FP16"; do
    echo "S16=$s | $c | $(FFG_S16=$s timeout 120 python scripts/k2_time.py $c 6 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
  for c in "2048 4 MIXED_EMULATED" "2048 1 MIXED_EMULATED" "4096 1 MIXED_EMULATED"; do
    echo "S16=$s | pair $c | $(FFG_WIDE=0 FFG_S16=$s timeout 120 python scripts/k2_time.py $c 4 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done; done 2>&1 | tee gpurun_out/s16sel.log
