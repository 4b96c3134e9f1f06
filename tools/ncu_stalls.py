"""Aggregate per-SASS-instruction warp-stall samples of an ncu --page source
--csv --print-source sass export.  usage: python tools/ncu_stalls.py src.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
per = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {c: int(r[ix[c]] or 0) for c in stall_cols}
    tot.update(st)
    op = r[ix["Source"]].split()[0:2]
    per.append((s, r[ix["Address"]], r[ix["Source"]][:90], max(st, key=st.get) if s else ""))
allс = sum(tot.values())
print("total samples", allс)
for k, v in tot.most_common(12):
    print(f"  {k:28s} {v:8d} {100*v/allс:5.1f}%")
per.sort(reverse=True)
for s, a, src, why in per[:top]:
    print(f"{s:7d} {100*s/allс:5.1f}% {a} {src:90s} {why}")
