"""Aggregate an ncu gpu__time_duration launch list by kernel name (total us, count)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Metric Name")
tot, cnt = collections.defaultdict(float), collections.defaultdict(int)
for r in rows[start + 1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
    name = r[ki].split("(")[0][:70]
    tot[name] += v
    cnt[name] += 1
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k]:10.1f} us  {cnt[k]:4d}x  {k}")
print(f"{sum(tot.values()):10.1f} us  total")
