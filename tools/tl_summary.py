"""Per-kernel totals of one ordered launch timeline (tools/ncu_timeline.py output) between two markers."""
import re, sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
a, b = sys.argv[2], sys.argv[3]
on = False; agg = defaultdict(lambda: [0, 0.0]); tot = 0
for l in lines:
    f = l.split(None, 3)
    if len(f) < 4: continue
    name = f[3]
    if not on and a in name: on = True
    elif on and b in name: break
    if on:
        key = re.sub(r"\s+\(\d+, \d+, \d+\)$", "", name)
        agg[key][0] += 1; agg[key][1] += float(f[1]); tot += float(f[1])
print(f"total {tot/1e3:.2f} ms")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{us/1e3:8.2f} ms n={n:4d} {us/n:8.1f} us  {k}")
