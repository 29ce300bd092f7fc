"""Development helper: sum the per-call '[positive]' lines of an SLM_POS_LOG=1 run (stdin)."""
import re, sys
keys = ("total", "lg", "alloc", "small1", "ginit", "gcta")
acc = {k: 0.0 for k in keys}; n = 0; rest = []
for line in sys.stdin:
    m = re.search(r"\| ([\d.]+) ms: lg ([\d.]+) alloc ([\d.]+) small1 ([\d.]+) ginit ([\d.]+) gcta ([\d.]+)", line)
    if not m:
        continue
    n += 1
    for k, v in zip(keys, m.groups()):
        acc[k] += float(v)
    rest.append(float(m.group(1)))
print("calls", n, {k: round(v, 1) for k, v in acc.items()})
print("first 5", rest[:5], "max", max(rest) if rest else 0)
