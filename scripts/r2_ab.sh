#!/bin/bash
# A/B of two library builds, alternating: $1 = variant name under lib/var (A), default build (B)
mkdir -p gpurun_out
A=paper_2605_08523_b200/lib/var/$1.so
shift
for r in 1 2 3; do for lib in A B; do
  L=""; [ $lib = A ] && L=$A
  for c in "$@"; do
    echo "$lib $c $(FFG_LIB_PATH=$L timeout 120 python scripts/k2_time.py $c 10 | sed 's/.*k2_ms_median": \([0-9.]*\).*/\1/')"
  done
done; done 2>&1 | tee gpurun_out/ab.log
python3 - <<'PY'
import collections
d=collections.defaultdict(list)
for l in open('gpurun_out/ab.log'):
    p=l.split()
    try: d[(p[0],' '.join(p[1:-1]))].append(float(p[-1]))
    except: pass
for k in sorted(set(c for _,c in d)):
    a=min(d[('A',k)]); b=min(d[('B',k)])
    print(f"{k:28s} A {a:8.4f}  B {b:8.4f}  B/A {b/a:.3f}")
PY
