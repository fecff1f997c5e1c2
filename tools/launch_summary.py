"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
for r in rows[1:]:
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:5d} {v[1]:9.3f} ms {100 * v[1] / tot:5.1f}%  {k}")
