#!/bin/bash
O=gpurun_out
: > $O/exp3.txt
for g in 4 8 16; do for ks in 8 16; do
  echo "G=$g KSTEP=$ks" >> $O/exp3.txt
  FFG_GROUP=$g FFG_NORMAL_KSTEP=$ks FFG_WIDE=1 MODES=MIXED_EMULATED timeout 120 python scripts/wide_check.py 1024x16 >> $O/exp3.txt 2>&1
done; done
for g in 16 32 64 128 512; do
  echo "G=$g" >> $O/exp3.txt
  FFG_GROUP=$g FFG_WIDE=1 timeout 200 python scripts/wide_check.py 512x512 >> $O/exp3.txt 2>&1
done
echo "pair 512x512" >> $O/exp3.txt
FFG_WIDE=0 timeout 200 python scripts/wide_check.py 512x512 >> $O/exp3.txt 2>&1
for ks in 8 16; do
  echo "KSTEP=$ks big" >> $O/exp3.txt
  FFG_NORMAL_KSTEP=$ks FFG_WIDE=1 timeout 300 python scripts/wide_check.py 4096x1 8192x1 >> $O/exp3.txt 2>&1
done
echo "pair big" >> $O/exp3.txt
FFG_WIDE=0 timeout 300 python scripts/wide_check.py 8192x1 >> $O/exp3.txt 2>&1
