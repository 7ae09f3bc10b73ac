"""Per-kernel registers / spills from the ptxas -v log of `make lib` (paper_2605_08523_b200/lib/ptxas.log)."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2605_08523_b200/lib/ptxas.log").read().splitlines()
cur = None
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and "Function properties" not in line:
        st, ld = m.group(2), m.group(3)
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        print(f"{cur[:70]:70s} regs {m2.group(1):>4s}  spill st {st:>4s} ld {ld:>4s}")
        cur = None
