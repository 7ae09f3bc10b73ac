"""Where a kernel's local-memory spills are: STL/LDL per source line, from `nvdisasm -g` output.

    nvdisasm -g lib.cubin > x.sass; python scripts/sass_spills.py x.sass <kernel-substring>
"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
key = sys.argv[2]
inside, cur, stats = False, None, {}
for l in lines:
    if l.startswith(".text."):
        inside = key in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"\b(STL|LDL)(\.\w+)*\s", l)
    if m:
        stats.setdefault(cur, [0, 0])[0 if m.group(1) == "STL" else 1] += 1
for k, v in sorted(stats.items(), key=lambda x: (str(x[0][0]), x[0][1])):
    print(f"{k[0]}:{k[1]}  STL {v[0]}  LDL {v[1]}")
