#!/bin/bash
# round-2 evidence: GPU tests, smoke, bench line, launch list, config sweep
O=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > $O/r2f_pytest.log 2>&1; echo "rc=$?" >> $O/r2f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2f_smoke.log 2>&1
timeout 600 python bench.py > $O/r2f_bench.json 2> $O/r2f_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/r2f_launches.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 1800 python scripts/config_sweep.py --out $O/r2f_configs.json > $O/r2f_sweep.log 2>&1
echo done
