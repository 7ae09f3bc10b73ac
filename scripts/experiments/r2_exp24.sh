#!/bin/bash
O=gpurun_out
: > $O/exp24.txt
for lib in default var/k1w8 var/k1w2; do
  if [ $lib = default ]; then L=""; else L="paper_2605_08523_b200/lib/$lib.so"; fi
  env ${L:+FFG_LIB_PATH=$L} timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:rescale -c 4 --csv python scripts/profile_step.py > $O/exp24_$(basename $lib).csv 2>/dev/null
  echo "$lib" >> $O/exp24.txt; grep -E "gpu__time|dram__bytes" $O/exp24_$(basename $lib).csv | tail -3 | cut -d, -f13- >> $O/exp24.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "spectral or golden or ragged or bench_config" >> $O/exp24.txt 2>&1
