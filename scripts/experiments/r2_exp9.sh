#!/bin/bash
O=gpurun_out
for ks in 8 16; do FFG_NORMAL_KSTEP=$ks timeout 300 python scripts/wide_check.py 1024x16 2048x4 4096x1 8192x1 > $O/exp9_k$ks.txt 2>&1; done
FFG_WIDE=0 timeout 300 python scripts/wide_check.py 1024x16 2048x4 4096x1 8192x1 > $O/exp9_pair.txt 2>&1
