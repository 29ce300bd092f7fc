"""Markdown table of one `ncu --set full` capture (raw page): per kernel time, DRAM bytes,
hit rates, occupancy, issue activity, registers, instructions, L1/L2 throughput.
usage: python tools/ncu_table.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
cols = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 thru %"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp inst")]
ix = [(h.index(c), name) for c, name in cols if c in h]
print("| kernel | " + " | ".join(n for _, n in ix) + " |")
print("|---" * (len(ix) + 1) + "|")
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    vals = []
    for i, _ in ix:
        u = units[i]
        v = r[i]
        try:
            f = float(v.replace(",", ""))
            v = f"{f:.4g} {u}".strip()
        except ValueError:
            pass
        vals.append(v)
    print(f"| `{name}` | " + " | ".join(vals) + " |")
