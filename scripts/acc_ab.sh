#!/bin/bash
# accuracy + K2 timing per library variant: bash scripts/acc_ab.sh lib_a.so lib_b.so ...
for L in "$@"; do
  export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/$L
  timeout 300 python scripts/accuracy_report.py MIXED_EMULATED 2>&1 | grep WORST | sed "s/^/$L /"
  timeout 120 python scripts/k2_variants.py 1024x16 512x64 4096x1 2>&1 | grep MIXED | sed "s/^.*\] //" | sed "s/^/$L /"
done
