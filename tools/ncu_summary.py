"""Summarise an ncu report: key metrics, stall reasons, top source lines."""
import csv, io, subprocess, sys

def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout

def details(rep, kregex):
    out = run([rep, "--page", "details", "--csv", "-k", f"regex:{kregex}"])
    rows = list(csv.reader(io.StringIO(out)))
    if not rows: return
    h = rows[0]
    si, mi, ui, vi = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    ki = h.index("Kernel Name")
    seen = set()
    for r in rows[1:]:
        key = (r[ki][:40], r[si], r[mi])
        if key in seen: continue
        seen.add(key)
        if r[si] in ("GPU Speed Of Light Throughput", "Occupancy", "Warp State Statistics", "Memory Workload Analysis", "Compute Workload Analysis", "Launch Statistics", "Scheduler Statistics"):
            print(f"{r[ki][:30]:30s} | {r[si][:26]:26s} | {r[mi]:55s} {r[vi]} {r[ui]}")

def source(rep, kregex, top=25):
    out = run([rep, "--page", "source", "--csv", "-k", f"regex:{kregex}", "--print-source", "sass,cuda"]) 
    print(out[:200])

if __name__ == "__main__":
    details(sys.argv[1], sys.argv[2])
