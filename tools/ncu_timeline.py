"""Ordered launch list from an `ncu --metrics gpu__time_duration.sum --csv`
log: one line per launch (index, us, short kernel name, grid), optionally
from the n-th occurrence of a marker kernel on (one call of a repeated step)."""
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, gi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Grid Size")
ui = h.index("Metric Unit")
out = []
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*\)$", "", r[ki]).replace("void ", "").replace("ppc::", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"<unnamed>::", "", name)
    v = float(r[vi].replace(",", ""))
    us = v / 1e3 if r[ui] == "ns" else (v if r[ui] in ("us", "usecond") else v * 1e3)
    out.append((us, name[:90], r[gi]))
marker = sys.argv[2] if len(sys.argv) > 2 else None
nth = int(sys.argv[3]) if len(sys.argv) > 3 else 1
start = 0
if marker:
    seen = 0
    for i, (_, n, _) in enumerate(out):
        if marker in n:
            seen += 1
            if seen == nth:
                start = i
                break
tot = 0.0
for i, (us, n, g) in enumerate(out[start:], start):
    tot += us
    print(f"{i:5d} {us:10.1f} {tot/1e3:9.2f}  {n}  {g}")
