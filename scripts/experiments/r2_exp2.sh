#!/bin/bash
O=gpurun_out
FFG_WIDE=1 timeout 300 python scripts/wide_check.py 256x1 > $O/exp2_wide.txt 2>&1
echo "rc=$?" >> $O/exp2_wide.txt
FFG_WIDE=1 timeout 600 python scripts/wide_check.py >> $O/exp2_wide.txt 2>&1
echo "rc=$?" >> $O/exp2_wide.txt
FFG_WIDE=0 timeout 600 python scripts/wide_check.py > $O/exp2_pair.txt 2>&1
