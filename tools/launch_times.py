"""Mean device time per kernel from an ncu --csv launch list (tools/launch_times.py f.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = {}
for r in rows[i + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    tot.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:60]:60s} n={len(v):3d} mean_us={sum(v) / len(v):9.1f}")
