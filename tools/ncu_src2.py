"""Per-kernel summary of an `ncu --page source --csv --print-source sass` dump: the sampled
stall hot spots of one function (the dump lists every function of the module)."""
import csv
import sys
from collections import Counter

path, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
sect, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur and pat in cur and hdr:
        sect.append(r)
if not sect:
    sys.exit("no such kernel")
ix = {h: i for i, h in enumerate(hdr)}
print(hdr)
samp = [(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r) for r in sect]
tot = sum(s for s, _ in samp)
print(f"{len(sect)} SASS lines, {tot:.0f} samples")
ops = Counter()
for s, r in samp:
    t = r[ix["Source"]].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    ops[op.split(".")[0]] += s
print("samples by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in ops.most_common(14)))
for s, r in sorted(samp, key=lambda x: -x[0])[:top]:
    print(f"{r[0][-5:]} {s:7.0f} {100*s/tot:5.1f}%  {r[ix['Source']].strip()[:90]}")

# stall reasons overall and for the hottest lines
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
totals = {h: sum(float(r[ix[h]] or 0) for r in sect) for h in st}
tt = sum(totals.values())
print("stalls:", ", ".join(f"{k[6:]} {100*v/tt:.1f}%" for k, v in sorted(totals.items(), key=lambda x: -x[1])[:10]))
ie = sum(float(r[ix["Instructions Executed"]] or 0) for r in sect)
print(f"warp instructions executed {ie:.4g}")
