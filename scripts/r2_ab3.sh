#!/bin/bash
# A/B/C of control-warp register budgets in the 16-worker pair kernel (FFG_R_CTL 40 default, 48, 56)
for r in 1 2 3; do for lib in default ctl48 ctl56; do
  L=""; [ $lib != default ] && L=paper_2605_08523_b200/lib/var/$lib.so
  for c in "1024 1 MIXED_EMULATED" "256 1 MIXED_EMULATED" "1024 4 MIXED_EMULATED" "1024 1 BF16" "512 64 MIXED_EMULATED"; do
    echo "$lib | $c | $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py $c 10 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done; done 2>&1 | tee gpurun_out/ab3.log
python3 - <<'PY'
import collections
d=collections.defaultdict(list)
for l in open('gpurun_out/ab3.log'):
    p=[x.strip() for x in l.split('|')]
    try: d[(p[0],p[1])].append(float(p[2]))
    except: pass
for c in sorted(set(k[1] for k in d)):
    print(f"{c:24s}", "  ".join(f"{lib} {min(d[(lib,c)]):.4f}" for lib in ("default","ctl48","ctl56")))
PY
