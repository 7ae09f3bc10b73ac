#!/bin/bash
# per-layer cost of each K2 kernel by layer type (timing only: all layers exact / none exact)
O=gpurun_out
: > $O/exp27.txt
for w in 0 1; do for x in 0 10 30; do
  echo "wide=$w exact=$x" >> $O/exp27.txt
  FFG_WIDE=$w FFG_EXACT_DRAIN_LAYERS=$x timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 10 >> $O/exp27.txt 2>&1
  FFG_WIDE=$w FFG_EXACT_DRAIN_LAYERS=$x FFG_NORMAL_KSTEP=16 timeout 120 python scripts/k2_time.py 1024 16 MIXED_EMULATED 10 >> $O/exp27.txt 2>&1
done; done
