#!/bin/bash
O=gpurun_out
: > $O/exp17.txt
for f in 2 4 6 8; do
  echo "FIRST=$f" >> $O/exp17.txt
  FFG_FIRST_KBLOCKS=$f FFG_WIDE=1 MODES=MIXED_EMULATED timeout 300 python scripts/wide_check.py 1024x16 1024x1 4096x1 >> $O/exp17.txt 2>&1
done
FFG_WIDE=1 timeout 900 python scripts/accuracy_sweep.py FFG_FIRST_KBLOCKS=2 FFG_FIRST_KBLOCKS=6 FFG_FIRST_KBLOCKS=8 > $O/exp17_acc.jsonl 2>&1
