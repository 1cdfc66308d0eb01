"""Summarise an ncu --page source --print-source=sass CSV: stall totals and
the top instructions per stall reason (used to write profiles/*.md)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
seen = set()
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] in seen or not r[0].startswith("0x"):
        continue
    seen.add(r[0])
    data.append(r)
tot = defaultdict(float)
for r in data:
    for c in stall_cols:
        try:
            tot[c] += float(r[idx[c]] or 0)
        except ValueError:
            pass
allsum = sum(tot.values())
print("stall totals:")
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:28s} {v:8.0f} {100 * v / allsum:5.1f}%")
want = sys.argv[2:] or ["stall_long_sb"]
for w in want:
    print(f"top instructions for {w}:")
    ranked = sorted(data, key=lambda r: -float(r[idx[w]] or 0))[:12]
    for r in ranked:
        print(f"  {float(r[idx[w]] or 0):7.0f} {r[0][-5:]} {r[1].strip()}")
