"""Summarise an ncu launch list with several metrics (time, dram read/write)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
cur, order = {}, []
for r in rows[start + 1:]:
    key = (r[0], r[ki][:34])
    if key not in cur:
        cur[key] = {}
        order.append(key)
    cur[key][r[mi].split("__")[1]] = float(r[vi].replace(",", ""))
for k in order[-n:]:
    d = cur[k]
    print(f"{k[0]:>4} {k[1]:34s} {d.get('time_duration.sum', 0) / 1e3:8.1f} us  rd {d.get('bytes_read.sum', 0) / 1e6:7.1f} MB"
          f"  wr {d.get('bytes_write.sum', 0) / 1e6:7.1f} MB")
