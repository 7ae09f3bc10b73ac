#!/bin/bash
# config 4 BF16 / FP32E: DRAM and L2 traffic of one K2 launch vs group size (is the group L2-resident?)
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum"
for mode in BF16 MIXED_EMULATED; do for g in 5 10 20 30; do
  echo "== $mode G=$g"
  FFG_GROUP=$g N=512 B=512 STEPS=1 MODE=$mode timeout 300 ncu --metrics $M --clock-control none -k regex:mlsp2 -c 1 --csv python scripts/profile_step.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done; done 2>&1 | tee gpurun_out/cfg4_dram.log
for n in 1024; do for g in 4 8 16; do
  echo "== bench N=1024 FP32E G=$g"
  FFG_GROUP=$g N=1024 B=16 STEPS=1 timeout 300 ncu --metrics $M --clock-control none -k regex:mlsp2 -c 1 --csv python scripts/profile_step.py 2>&1 | grep -E '"(gpu__|dram__|lts__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done; done 2>&1 | tee -a gpurun_out/cfg4_dram.log
