#!/bin/bash
# One GPU round trip: gated tests, bench line, launch list and one K2 full capture.
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench.json 2> $O/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/launches.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_pair -s 1 -c 1 -o $O/k2_full -f python scripts/profile_step.py > $O/ncu_full.log 2>&1
echo done
