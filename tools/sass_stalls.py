"""Top SASS stall sites from `ncu -i rep --page source --csv --print-source sass`.
usage: python tools/sass_stalls.py sass.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ix = {k: h.index(k) for k in h}
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0 for c in cols}
lines = []
seen = set()
for r in rows[2:]:
    if r and r[0] in seen:
        continue  # the export can list an instruction twice
    if r:
        seen.add(r[0])
    if len(r) < len(h) or r[0] == "Address" or not r[ix["Warp Stall Sampling (All Samples)"]].isdigit():
        continue  # short rows, repeated headers (one block per kernel instance)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for c in cols:
        tot[c] += int(r[ix[c]] or 0)
    lines.append((s, r[ix["Address"]], r[ix["Source"]], {c: int(r[ix[c]] or 0) for c in cols}))
allv = sum(tot.values())
print("total samples", allv)
print({c[6:]: round(v / allv, 3) for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
for s, a, src, d in sorted(lines, key=lambda x: -x[0])[:top]:
    main = sorted(d.items(), key=lambda x: -x[1])[:2]
    print(f"{s:6d} {a} {src[:60]:60s} {[(k[6:], v) for k, v in main]}")
