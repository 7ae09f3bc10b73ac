#!/bin/bash
# A/B of K2 build variants: for each lib under paper_2605_08523_b200/lib/var, smoke parity then K2 timing.
# usage: bash scripts/ab_libs.sh "1024x16 4096x1 512x64" lib_a.so lib_b.so ...
cases=$1; shift
mkdir -p gpurun_out
for L in "$@"; do
  export FFG_LIB_PATH=paper_2605_08523_b200/lib/var/$L
  echo "=== $L"
  timeout 120 python scripts/smoke_small.py 2>&1 | grep -E "^(1024|512|100|384) |batch [05]|Error|error|Trace" | head -12
  timeout 240 python scripts/k2_variants.py $cases 2>&1 | grep -E "K2|rror" | sed "s/^/$L /"
done
