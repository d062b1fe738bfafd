"""Summarise an `ncu --page source --csv --print-source sass` dump: top
instructions by stall samples with their dominant stall reasons (dev tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = rows[2:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total samples", tot)
agg = {c: 0 for c in stall_cols}
for r in data:
    for c in stall_cols:
        agg[c] += int(r[ix[c]] or 0)
print("by reason:", sorted(((v, c) for c, v in agg.items() if v), reverse=True)[:10])
top = sorted(data, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols if int(r[ix[c]] or 0)), reverse=True)[:3]
    print(f"{s:7d} {100*s/tot:5.1f}% {r[0][-5:]} {r[1].strip()[:60]:60s} exec={r[ix['Instructions Executed']]} {reasons}")
