#!/bin/bash
# host-path (e2e) throughput vs pipeline chunk count, plus raw PCIe copy rates
python scripts/pcie_probe.py
for c in 1 2 4 8; do
  FFG_E2E_CHUNKS=$c timeout 200 python bench.py --steps 30 2>/dev/null > /tmp/b_$c.json
  python - "$c" <<'PY'
import json, sys
d = json.load(open(f"/tmp/b_{sys.argv[1]}.json"))
print("chunks", sys.argv[1], round(d["value"]), round(d["e2e"]["value"]))
PY
done
