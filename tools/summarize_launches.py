"""Summarise an ncu launch list of bench.py's timed region (tools/prof.sh): per-kernel time
and DRAM bytes for one sweep, and write profiles/plan_sweep_traffic.json.
usage: python tools/summarize_launches.py gpurun_out/launches_TAG.csv TAG [steps] [write]"""
import collections, csv, json, os, sys

path, tag = sys.argv[1], sys.argv[2]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
per = collections.OrderedDict()
for r in rows[1:]:
    key = (int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0])
    v = float(r[ix["Metric Value"]])
    u = r[ix["Metric Unit"]]
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}.get(u, 1.0)
    per.setdefault(key, {})[r[ix["Metric Name"]]] = v * scale
agg = collections.OrderedDict()
for (i, name), m in per.items():
    a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot_t = sum(a[1] for a in agg.values())
tot_b = sum(a[2] + a[3] for a in agg.values())
lines = [f"launch list {os.path.basename(path)}: {len(per)} launches over {steps} timed sweeps "
         f"(cold-cache, serialised: compare shares)", "",
         "| kernel | launches/sweep | ms/sweep | share | DRAM read GB/sweep | DRAM write GB/sweep |",
         "|---|---|---|---|---|---|"]
for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{name}` | {n / steps:g} | {t / steps:.3f} | {100 * t / tot_t:.1f}% | "
                 f"{rd / steps / 1e9:.3f} | {wr / steps / 1e9:.3f} |")
lines.append(f"| total | {len(per) / steps:g} | {tot_t / steps:.3f} | 100% | | |")
print("\n".join(lines))
out = {"round": tag, "workload": "c5_rmat24", "dram_bytes_per_sweep": int(tot_b / steps),
       "method": f"ncu --profile-from-start off (bench.py timed region, {steps} sweeps): sum of "
                 "dram__bytes_read.sum + dram__bytes_write.sum over every launch / sweeps",
       "source": os.path.basename(path)}
if len(sys.argv) > 4 and sys.argv[4] == "write":
  json.dump(out, open(os.path.join(os.path.dirname(__file__), "..", "profiles",
                                 "plan_sweep_traffic.json"), "w"), indent=1)
