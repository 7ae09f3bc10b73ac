#!/bin/bash
O=gpurun_out
for t in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_small.py > $O/r2b_sanitizer_$t.log 2>&1; echo "$t rc=$?" >> $O/r2b_sanitizer_$t.log
done
N=4096 B=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/wide4096 -f python scripts/profile_step.py > $O/ncu_w4096.log 2>&1
