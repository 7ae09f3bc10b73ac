#!/bin/bash
# TMA multicast vs unicast operand streaming (scripts/mc_bench.cu) + L2 sectors per mode
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mc_bench scripts/mc_bench.cu -lcuda || exit 1
timeout 120 /tmp/mc_bench 2>&1 | tee gpurun_out/mc_bench.log

