#!/bin/bash
# evidence after the kernel-selection change (16-worker pair kernel up to N=2048, wide from N=4096):
# launch list + full K2 capture of the bench step, config sweep, bench line, smoke
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv --log-file $O/fc_launches.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_pair -s 1 -c 1 -o $O/fc_pair_full -f python scripts/profile_step.py > $O/fc_ncu.log 2>&1
timeout 2400 python scripts/config_sweep.py --out $O/fc_configs.json > $O/fc_sweep.log 2>&1
timeout 600 python bench.py > $O/fc_bench.json 2> $O/fc_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fc_smoke.log 2>&1
echo done
