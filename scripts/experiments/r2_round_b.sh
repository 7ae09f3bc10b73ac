#!/bin/bash
# bench line, launch list, K2 full capture, config sweep (wide kernel default)
O=gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 > $O/bench_b.json 2> $O/bench_b.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/launches_b.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_wide -s 1 -c 1 -o $O/k2_wide_full -f python scripts/profile_step.py > $O/ncu_full_b.log 2>&1
timeout 1500 python scripts/config_sweep.py --out $O/r2_configs_b.json > $O/sweep_b.log 2>&1
echo done
