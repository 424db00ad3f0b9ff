"""Print the hottest SASS lines (warp-stall samples) of an ncu --page source --csv dump."""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
h = r[1]
si = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
rows = []
for row in r[2:]:
    try:
        v = float(row[si] or 0)
    except ValueError:
        continue
    rows.append((v, row))
tot = sum(v for v, _ in rows) or 1
agg = {}
for v, row in rows:
    for i in stall_cols:
        try:
            agg[h[i]] = agg.get(h[i], 0) + float(row[i] or 0)
        except ValueError:
            pass
print("stall totals:", sorted(((k, round(v / tot * 100, 1)) for k, v in agg.items() if v), key=lambda kv: -kv[1])[:8])
rows.sort(key=lambda x: -x[0])
for v, row in rows[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(((h[i], float(row[i] or 0)) for i in stall_cols), key=lambda kv: -kv[1])[:2]
    print(f"{v / tot * 100:5.1f}% exec={row[ex]:>8s} {row[0]:>6s} {row[1][:80]:80s} {top}")
