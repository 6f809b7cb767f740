"""Stall samples per CUDA source line from an ncu report (mixed sass,cuda
source page): python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.StringIO(out)))
fname, res = None, []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 3 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        try:
            res.append((float(r[wi] or 0), float(r[ei] or 0), fname, int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
for w, e, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{w / tot * 100:5.1f}% samp {e / toti * 100:5.1f}% inst  {f}:{ln}  {src[:90]}")
