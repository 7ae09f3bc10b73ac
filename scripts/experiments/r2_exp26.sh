#!/bin/bash
O=gpurun_out
FFG_WIDE=0 MODES=MIXED_EMULATED,BF16 timeout 300 python scripts/wide_check.py 1024x16 1024x1 512x128 > $O/exp26.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q >> $O/exp26.txt 2>&1; echo "rc=$?" >> $O/exp26.txt
