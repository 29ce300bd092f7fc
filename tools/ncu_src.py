"""Summarise an `ncu --page source --csv --print-source sass` dump: totals, stall mix,
hottest instructions (by stall samples) and instruction-class counts."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data, seen = [], set()
for r in rows[2:]:   # the dump repeats the listing once per source view; keep one copy
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
def f(r, k):
    try: return float(r[ix[k]])
    except ValueError: return 0.0
tot_inst = sum(f(r, "Instructions Executed") for r in data)
tot_samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(rows[0][1][:100])
print(f"warp instructions executed {tot_inst:.4g}, stall samples {tot_samp:.0f}")
st = collections.Counter()
for r in data:
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            st[h] += f(r, h)
print("stalls:", ", ".join(f"{k[6:]} {100*v/max(tot_samp,1):.1f}%" for k, v in st.most_common(8)))
op = collections.Counter(); ops = collections.Counter()
for r in data:
    m = r[ix["Source"]].split()
    if not m: continue
    o = m[0] if not m[0].startswith("@") else m[1]
    op[o.split(".")[0]] += f(r, "Instructions Executed")
    ops[o.split(".")[0]] += f(r, "Warp Stall Sampling (All Samples)")
print("by opcode (inst%, samples%):")
for k, v in op.most_common(25):
    print(f"  {k:10s} {100*v/tot_inst:5.1f}% {100*ops[k]/max(tot_samp,1):5.1f}%")
import signal; signal.signal(signal.SIGPIPE, signal.SIG_DFL)
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
print("hottest:")
for r in top:
    print(f"  {r[ix['Address']][-5:]} {f(r,'Warp Stall Sampling (All Samples)'):6.0f} {f(r,'Instructions Executed'):10.0f}  {r[ix['Source']].strip()[:70]}")
