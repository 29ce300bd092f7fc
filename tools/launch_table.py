"""Per-kernel totals of an ncu launch-list CSV (gpu__time_duration.sum): python tools/launch_table.py f.csv"""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]]); u = r[ix["Metric Unit"]]
    v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
    a = agg[r[ix["Kernel Name"]].split("(")[0][:60]]
    a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{t:8.3f} ms {100*t/tot:5.1f}% {n:4d}x  {k}")
