"""Hot CUDA lines and SASS instructions from
`ncu -i X --page source --csv --print-source sass,cuda -k regex:K > out.csv`."""
import csv, sys

def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0

def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    lines, sass, cur = [], [], None
    for r in rows[hi + 1:]:
        if len(r) < len(h) - 3:
            continue
        if r[0]:
            cur = (r[0], r[1].strip())
            lines.append((f(r[wi]), f(r[ei]), cur))
        else:
            sass.append((f(r[wi]), f(r[ei]), cur, r[3].strip()))
    tot = sum(x[0] for x in sass) or 1.0
    print(f"stall samples {tot:.0f}")
    for w, e, (ln, src) in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"{100 * w / tot:5.1f}% L{ln:>4s} inst {e:9.0f}  {src[:90]}")
    print("--- SASS")
    for w, e, cur, ins in sorted(sass, key=lambda x: -x[0])[:top]:
        print(f"{100 * w / tot:5.1f}% L{cur[0] if cur else '?':>4s} {ins[:70]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
