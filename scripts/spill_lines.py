"""STL/LDL per innermost kernel-source line of one kernel (nvdisasm -gi output; measurement script).

    cuobjdump -xelf all lib.so; nvdisasm -gi x.cubin > x.sass; python scripts/spill_lines.py x.sass <kernel-substring>
"""
import collections
import re
import sys

inside, cur, seq = False, None, False
st, ld = collections.Counter(), collections.Counter()
for l in open(sys.argv[1]):
    if l.startswith(".text."):
        inside = sys.argv[2] in l
        continue
    if not inside:
        continue
    if l.lstrip().startswith("//## File"):
        locs = [f'{f.split("/")[-1]}:{n}' for f, n in re.findall(r'"([^"]+)", line (\d+)', l)]
        own = [x for x in locs if x.startswith(("k2_", "epilogue"))]
        if not seq or cur is None or not cur.startswith(("k2_", "epilogue")):
            cur = own[0] if own else locs[0]
        seq = True
        continue
    seq = False
    if re.search(r"\bSTL", l):
        st[cur] += 1
    if re.search(r"\bLDL", l):
        ld[cur] += 1
for k in sorted(set(st) | set(ld), key=lambda k: -(st[k] + ld[k]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{k:28s} STL {st[k]:4d}  LDL {ld[k]:4d}")
