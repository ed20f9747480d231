"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
for r in rows[start + 1:]:
    v = float(r[vi].replace(",", ""))
    if r[ui] == "ns":
        v /= 1e3
    elif r[ui] == "ms":
        v *= 1e3
    print(f"{r[0]:>4} {v:10.2f} us  {r[ki][:90]}")
