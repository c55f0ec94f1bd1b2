"""Summarize an ncu --page source --csv --print-source sass export: the hottest
SASS instructions of the first kernel with their dominant stall reasons, and the
instruction mix. Usage: ncu -i rep --page source --csv --print-source sass | python ncu_sass_hot.py [kernel_index]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(sys.stdin))
want = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        kernels.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None and r:
        cur[2].append(r)
name, hdr, rs = kernels[want]
idx = {h: j for j, h in enumerate(hdr)}
S = idx["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S] or 0) for r in rs) or 1
print(name[:120])
print("stall totals:", ", ".join(f"{h[6:]} {100*sum(int(r[idx[h]] or 0) for r in rs)/tot:.1f}%"
                                   for h in stalls if sum(int(r[idx[h]] or 0) for r in rs) > 0.01 * tot))
for r in sorted(rs, key=lambda r: -int(r[S] or 0))[:20]:
    top = sorted(((int(r[idx[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{100*int(r[S])/tot:5.1f}%  {r[idx['Source']].strip()[:60]:60s} {top}")
c = Counter()
for r in rs:
    src = r[idx["Source"]].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    c[op.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
print("mix:", c.most_common(14))
