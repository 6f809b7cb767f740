"""Print an ncu launch list (gpu__time_duration.sum CSV) as an ordered table
with each kernel's share of the total."""
import csv, re, sys

def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    out = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.match(r"(?:void )?(?:srlu::)?([A-Za-z0-9_:]+)", name)
        short = m.group(1) if m else name[:40]
        t = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "ns":
            t /= 1e3
        elif r["Metric Unit"] == "ms":
            t *= 1e3
        out.append((short[:48], r["Stream"], r["Grid Size"], r["Block Size"], t))
    return out

if __name__ == "__main__":
    rows = load(sys.argv[1])
    tot = sum(r[4] for r in rows)
    for s, st, g, b, t in rows:
        print(f"{s:48s} s{st:>3s} {g:>14s} {b:>12s} {t:9.1f} us {100 * t / tot:5.1f}%")
    print(f"{'total':48s} {tot:9.1f} us over {len(rows)} launches")
