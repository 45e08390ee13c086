"""Per-kernel registers / spills from `nvcc -Xptxas -v` output on stdin (filter: argv[1] regex)."""
import re
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(2)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if pat is None or pat.search(cur):
            print(f"{m.group(1):>4} regs  spill {spill:>4}  {cur}")
        cur = None
