#!/bin/bash
# ncu --set full of one K2 launch: config 4 (512 x N=512) FP32E and BF16, and the wide kernel at the bench config
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -k regex:mlsp2 -c 1"
N=512 B=512 STEPS=1 MODE=MIXED_EMULATED timeout 900 $NCU -o gpurun_out/r2_cfg4_fp32e -f python scripts/profile_step.py > gpurun_out/ncu_cfg4_a.log 2>&1
N=512 B=512 STEPS=1 MODE=BF16 timeout 900 $NCU -o gpurun_out/r2_cfg4_bf16 -f python scripts/profile_step.py > gpurun_out/ncu_cfg4_b.log 2>&1
FFG_WIDE=1 N=1024 B=16 STEPS=1 MODE=MIXED_EMULATED timeout 900 $NCU -o gpurun_out/r2_wide_n1024 -f python scripts/profile_step.py > gpurun_out/ncu_wide1024.log 2>&1
tail -3 gpurun_out/ncu_*.log
