#!/bin/bash
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file $O/r2g_launches.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 2000 python -m pytest tests -m gpu -q > $O/r2g_pytest.log 2>&1; echo "rc=$?" >> $O/r2g_pytest.log
