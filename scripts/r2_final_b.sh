#!/bin/bash
# round-2 final evidence: tests, smoke, bench line, launch list, K2 capture, config sweep, sanitizers
O=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > $O/fb_pytest.log 2>&1; echo "rc=$?" >> $O/fb_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fb_smoke.log 2>&1
timeout 600 python bench.py > $O/fb_bench.json 2> $O/fb_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv --log-file $O/fb_launches.csv python scripts/profile_step.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlsp2_pair -s 1 -c 1 -o $O/fb_pair_full -f python scripts/profile_step.py > $O/fb_ncu.log 2>&1
timeout 2400 python scripts/config_sweep.py --out $O/fb_configs.json > $O/fb_sweep.log 2>&1
for t in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_small.py > $O/fb_sanitizer_$t.log 2>&1; echo "$t rc=$?" >> $O/fb_sanitizer_$t.log
done
echo done
