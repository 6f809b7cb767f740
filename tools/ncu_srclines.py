"""Per-CUDA-source-line instruction and stall-sample shares of one kernel in
an ncu --set full --import-source report:
  python tools/ncu_srclines.py report.ncu-rep kernel_regex [top] [sort=inst|samp]"""
import csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
key = sys.argv[4] if len(sys.argv) > 4 else "inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
fname, hdr, res = None, None, []
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname, hdr = r[1].split("/")[-1], None
    elif len(r) > 3 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        wi, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        try:
            res.append((float(r[wi] or 0), float(r[ei] or 0), fname, int(r[0]), r[1].strip()))
        except ValueError:
            pass
ts = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for w, e, f, ln, src in sorted(res, key=lambda x: -(x[1] if key == "inst" else x[0]))[:top]:
    print(f"{w / ts * 100:5.1f}% samp {e / ti * 100:5.1f}% inst  {f}:{ln}  {src[:80]}")
