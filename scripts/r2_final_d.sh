#!/bin/bash
# round-end evidence on the final build: GPU tests, smoke, bench line, compute-sanitizer
O=gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > $O/fd_pytest.log 2>&1; echo "rc=$?" >> $O/fd_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/fd_smoke.log 2>&1
timeout 600 python bench.py > $O/fd_bench.json 2> $O/fd_bench.err
timeout 600 python bench.py --impl reference > $O/fd_bench_ref.json 2> $O/fd_bench_ref.err
for t in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_small.py > $O/fd_sanitizer_$t.log 2>&1; echo "$t rc=$?" >> $O/fd_sanitizer_$t.log
done
echo done
