#!/bin/bash
# K2 time per layer vs L2-resident group size (FFG_GROUP)
for c in "$@"; do for g in 4 6 9 12 16 24 32 64; do
  FFG_GROUP=$g timeout 100 python scripts/k2_variants.py $c 2>&1 | grep -E "K2" | sed "s/^.*\] //" | sed "s/^/G=$g /"
done; done
