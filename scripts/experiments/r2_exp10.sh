#!/bin/bash
O=gpurun_out
timeout 300 python scripts/wide_check.py 1024x16 1024x64 512x128 > $O/exp10.txt 2>&1
FFG_WIDE=0 timeout 300 python scripts/wide_check.py 1024x64 >> $O/exp10.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_wide.log 2>&1; echo "rc=$?" >> $O/pytest_wide.log
