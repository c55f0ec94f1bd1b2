"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel (template args collapsed to the configuration): count, total ms, share."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    name = re.sub(r"\(ppc::GemmParams\)|\(.*\)$", "", name)
    name = name.replace("void ", "").replace("ppc::", "").replace("(anonymous namespace)::", "")
    v = float(r[vi].replace(",", ""))
    unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "ns"
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"total kernel time {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ms:10.3f} ms {100*ms/tot:5.1f}%  n={n:5d}  {name[:110]}")
