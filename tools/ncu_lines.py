"""Per-source-line instruction / stall totals from `ncu --page source --csv --print-source
cuda,sass` (interleaved listing: a row with a line number starts a source line, the
following rows with an address are its SASS).  usage: ncu_lines.py dump.csv [norm]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = None
line = None
acc = collections.OrderedDict()
src = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    if r[0]:
        line = int(r[0])
        src[line] = r[1]
        continue
    try:
        e = float(r[7] or 0); s = float(r[4] or 0)
    except ValueError:
        continue
    a = acc.setdefault(line, [0.0, 0.0])
    a[0] += e; a[1] += s
te = sum(v[0] for v in acc.values()); ts = sum(v[1] for v in acc.values())
print(f"total inst {te:.4g} ({te/norm:.1f} per unit), samples {ts:.0f}")
for l, (e, s) in acc.items():
    if e / te > 0.004 or s / max(ts, 1) > 0.01:
        print(f"{l:5d} {e/norm:8.1f} {100*e/te:5.1f}% {100*s/max(ts,1):5.1f}%  {src.get(l,'')[:80]}")
