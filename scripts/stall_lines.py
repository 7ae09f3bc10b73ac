"""Warp-stall samples of an ncu capture aggregated per source line (measurement script).

    ncu -i rep --page source --csv --print-source=sass > k.csv
    nvdisasm -gi lib.cubin > k.sass
    python scripts/stall_lines.py k.csv k.sass <kernel-substring> [top]
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
addr_s = {}
for r in rows[2:]:
    if len(r) <= isamp:
        continue
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    addr_s[a] = (float(r[isamp] or 0), {hdr[i]: float(r[i] or 0) for i in stall_cols})
base = min(addr_s) if addr_s else 0  # ncu lists absolute addresses
addr_s = {a - base: v for a, v in addr_s.items()}
# address -> source line from nvdisasm -g
key = sys.argv[3]
line_of = {}
inside, cur, in_seq = False, None, False
for l in open(sys.argv[2]):
    if l.startswith(".text."):
        inside = key in l
        continue
    if not inside:
        continue
    if l.lstrip().startswith("//## File"):
        # nvdisasm -gi: "file, line N inlined at file, line M" -- attribute to the kernel's own line
        locs = [f'{f.split("/")[-1]}:{n}' for f, n in re.findall(r'"([^"]+)", line (\d+)', l)]
        own = [x for x in locs if x.startswith(("k2_", "epilogue"))]
        if not in_seq or cur is None or not cur.startswith(("k2_", "epilogue")):
            cur = own[0] if own else locs[0]  # the innermost kernel-file line of the inline chain
        in_seq = True
        continue
    in_seq = False
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
tot = defaultdict(float)
why = defaultdict(lambda: defaultdict(float))
for a, (s, st) in addr_s.items():
    k = line_of.get(a, "?")
    tot[k] += s
    for n, v in st.items():
        why[k][n] += v
T = sum(tot.values())
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    reasons = sorted(why[k].items(), key=lambda x: -x[1])[:3]
    print(f"{k:28s} {100 * v / T:5.1f}%  " + "  ".join(f"{n[6:]}={100 * x / T:.1f}" for n, x in reasons))
