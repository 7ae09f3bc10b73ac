#!/bin/bash
O=gpurun_out
: > $O/exp21.txt
for c in 1 2 4; do
  FFG_E2E_CHUNKS=$c timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu > $O/b21_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b21_$c.json')); print('chunks=$c', d['value'], d['e2e']['value'])" >> $O/exp21.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "async or host_path or two_streams" >> $O/exp21.txt 2>&1
