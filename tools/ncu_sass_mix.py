"""Instruction mix and hottest SASS lines of an ncu report (needs --import-source on).
    python tools/ncu_sass_mix.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h)]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[ie] or 0) for x in rows)
tst = sum(int(x[st] or 0) for x in rows) or 1
print("total warp instructions", tot)
c = Counter()
for x in rows:
    t = x[src].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    c[op.split(".")[0]] += int(x[ie] or 0)
for k, v in c.most_common(22):
    print(f"  {k:12s} {v:12d} {v / tot * 100:5.1f}%")
print("hottest lines by stall samples:")
for x in sorted(rows, key=lambda x: -int(x[st] or 0))[:top_n]:
    print(f"  {int(x[st] or 0) / tst * 100:5.1f}% {int(x[ie] or 0):11d}  {x[src].strip()[:90]}")
