"""Fold the comm_balance.py ncu launch list into per-plan Q^max_p vs Q^sum_p/p
(DRAM and L2 bytes per worker) -> JSON + a table (§8f-f3)."""
import csv, collections, json, sys

layout = json.load(open(sys.argv[1]))
rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10]
hdr = rows[0]
idi, mi, vi, ui = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[int(r[idi])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
ids = sorted(per)
L = layout["launches"]
assert len(ids) == len(L), (len(ids), len(L))
out = collections.defaultdict(lambda: collections.defaultdict(lambda: [0.0, 0.0, 0.0]))
for lid, rec in zip(ids, L):
    m = per[lid]
    w = out[(rec["p"], rec["plan"])][rec["worker"]]
    w[0] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    w[1] += m.get("lts__t_bytes.sum", 0)
    w[2] += 4 * (rec["n"] * rec["k"] + rec["k"] * rec["m"] + rec["n"] * rec["m"])
res = []
print(f"{'p':>2} {'plan':<10} {'DRAM Qmax':>10} {'Qsum/p':>10} {'ratio':>6} | {'L2 max/avg':>10} | {'surface max/avg':>15}")
for (p, plan), ws in sorted(out.items()):
    d = [v[0] for v in ws.values()]; l2 = [v[1] for v in ws.values()]; sf = [v[2] for v in ws.values()]
    row = {"p": p, "plan": plan, "dram_max": max(d), "dram_sum": sum(d), "dram_ratio": max(d) / (sum(d) / p),
           "l2_ratio": max(l2) / (sum(l2) / p), "surface_ratio": max(sf) / (sum(sf) / p),
           "dram_per_worker": d, "l2_per_worker": l2, "surface_per_worker": sf}
    res.append(row)
    print(f"{p:>2} {plan:<10} {max(d)/1e9:9.2f}G {sum(d)/p/1e9:9.2f}G {row['dram_ratio']:6.3f} | {row['l2_ratio']:10.3f} | {row['surface_ratio']:15.3f}")
json.dump({"n": layout["n"], "semiring": "minplus_sat32", "plans": res}, open(sys.argv[3], "w"), indent=1)
