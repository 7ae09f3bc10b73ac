#!/bin/bash
# register budgets: 16-worker control warps 56 / 64 (FFG_R_CTL); 8-warp variant (FFG_P_CTL/DRAIN/EPI) trades
for r in 1 2 3; do for lib in default ctl56 ctl64 v0a v0b; do
  L=""; [ $lib != default ] && L=paper_2605_08523_b200/lib/var/$lib.so
  for c in "1024 1 MIXED_EMULATED" "1024 16 MIXED_EMULATED" "1024 16 BF16" "512 512 MIXED_EMULATED"; do
    echo "$lib | $c | $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py $c 10 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done; done 2>&1 | tee gpurun_out/ab4.log
python3 - <<'PY'
import collections
d=collections.defaultdict(list)
for l in open('gpurun_out/ab4.log'):
    p=[x.strip() for x in l.split('|')]
    try: d[(p[0],p[1])].append(float(p[2]))
    except: pass
for c in sorted(set(k[1] for k in d)):
    print(f"{c:24s}", "  ".join(f"{lib} {min(d[(lib,c)]):.4f}" for lib in ("default","ctl56","ctl64","v0a","v0b") if d[(lib,c)]))
PY
