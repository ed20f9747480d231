"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[hi]
si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((float(r[si] or 0), r[0], r[src]))
    except (ValueError, IndexError):
        continue
tot = sum(d[0] for d in data) or 1
for s, a, t in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% {a} {t[:110]}")
