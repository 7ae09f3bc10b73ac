#!/bin/bash
# normal-layer chunk length (FFG_NORMAL_KSTEP 8 = default, 16): K2 time and the FP32E gates
for r in 1 2; do for k in 8 16; do
  for c in "1024 1 MIXED_EMULATED" "1024 16 MIXED_EMULATED" "512 512 MIXED_EMULATED" "4096 1 MIXED_EMULATED"; do
    echo "k=$k | $c | $(FFG_NORMAL_KSTEP=$k timeout 120 python scripts/k2_time.py $c 6 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done; done 2>&1 | tee gpurun_out/kstep.log
FFG_NORMAL_KSTEP=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -3
FFG_NORMAL_KSTEP=16 timeout 300 python scripts/accuracy_report.py 2>&1 | tail -12
