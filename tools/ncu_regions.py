"""Stall-reason breakdown of an ncu source-page CSV (SASS) by code region:
regions are split at the given hex address suffixes (or automatically by
0x800 blocks).  Usage: python tools/ncu_regions.py src.csv [addr ...]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ai, si, ei = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
f = lambda x: float(x.replace(",", "") or 0)
tot_i = sum(f(r[ei]) for r in data)
tot = {k: sum(f(r[h.index(k)]) for r in data) for k in reasons}
allsamp = sum(tot.values())
print("overall:", ", ".join(f"{k[6:]} {v / allsamp * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
cuts = [int(x, 16) for x in sys.argv[2:]]
reg = defaultdict(lambda: [0.0, defaultdict(float), None])
for r in data:
    a = int(r[ai], 16)
    key = sum(1 for c in cuts if (a & 0xfffff) >= c) if cuts else (a >> 11)
    reg[key][0] += f(r[ei])
    for k in reasons:
        reg[key][1][k] += f(r[h.index(k)])
    if reg[key][2] is None:
        reg[key][2] = r[ai][-5:] + " " + r[si][:40]
for key in sorted(reg):
    e, st, s = reg[key]
    samp = sum(st.values())
    if samp / allsamp < 0.01 and e / tot_i < 0.01:
        continue
    top = ", ".join(f"{k[6:]} {v / allsamp * 100:.1f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4])
    print(f"{s:48s} inst {e / tot_i * 100:5.1f}% samp {samp / allsamp * 100:5.1f}%  [{top}]")
