"""Summarise an `ncu --page source --csv --print-source sass` dump: stall samples by reason,
and the top instructions by samples (optionally within an address range).

    python tools/ncu_stalls.py dump.csv [lo_hex hi_hex] [top]
"""
import csv, sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
inst = []
base = int(data[0][ix["Address"]], 16)
for r in data:
    a = int(r[ix["Address"]], 16) - base
    if not (lo <= a < hi):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for h in reasons:
        v = r[ix[h]]
        if v:
            tot[h] += int(v)
    inst.append((s, a, r[ix["Source"]], {h: int(r[ix[h]]) for h in reasons if r[ix[h]] and int(r[ix[h]]) > 0}))
T = sum(tot.values())
print("total samples", T)
for h, v in tot.most_common():
    print(f"  {h:28s} {v:8d} {100 * v / max(T, 1):5.1f}%")
inst.sort(reverse=True)
for s, a, src, d in inst[:top]:
    dd = ", ".join(f"{k[6:]}={v}" for k, v in sorted(d.items(), key=lambda x: -x[1])[:3])
    print(f"{a:06x} {s:6d} {src[:60]:60s} {dd}")
