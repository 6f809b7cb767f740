"""Top SASS instructions by stall samples / executed instructions from an ncu source page CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
ai, si, wi, ei = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
def f(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
tot_w = sum(f(r[wi]) for r in data); tot_e = sum(f(r[ei]) for r in data)
print(f"total stall samples {tot_w:.0f}  instr executed {tot_e:.3e}")
key = wi if len(sys.argv) < 3 else ei
for r in sorted(data, key=lambda r: -f(r[key]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{f(r[wi])/max(tot_w,1)*100:5.1f}% samp {f(r[ei])/max(tot_e,1)*100:5.1f}% inst  {r[ai]}  {r[si][:90]}")
