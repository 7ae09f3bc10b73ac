#!/bin/bash
O=gpurun_out
timeout 300 python scripts/timeline_e2e.py > $O/tl_e2e2.txt 2>&1
: > $O/exp22.txt
for c in 1 2; do
  FFG_E2E_CHUNKS=$c timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu > $O/b22_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b22_$c.json')); print('chunks=$c', d['value'], d['e2e']['value'])" >> $O/exp22.txt
done
timeout 1500 python -m pytest tests -m gpu -q -x >> $O/exp22.txt 2>&1
