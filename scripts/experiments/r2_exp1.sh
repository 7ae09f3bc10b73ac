#!/bin/bash
# accuracy vs chunk length of the non-exact layers; K2 time vs group size (bench config)
O=gpurun_out
timeout 900 python scripts/accuracy_sweep.py FFG_NORMAL_KSTEP=8 FFG_NORMAL_KSTEP=16 FFG_NORMAL_KSTEP=32 FFG_NORMAL_KSTEP=4096 > $O/exp1_acc.jsonl 2>&1
for g in 2 3 4 5 6 8 16; do FFG_GROUP=$g timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 10; done > $O/exp1_group.jsonl 2>&1
for g in 8 16 32 64 128; do FFG_GROUP=$g timeout 120 python scripts/k2_time.py 512 512 MIXED_EMULATED 5; done >> $O/exp1_group.jsonl 2>&1
