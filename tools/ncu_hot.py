"""Summarise an `ncu --page source --csv --print-source sass` export: top SASS lines by
warp-stall samples, with their dominant stall reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ci = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(float(r[ci] or 0) for r in data)
agg = {}
for i in stall_cols:
    agg[h[i]] = sum(float(r[i] or 0) for r in data)
print("total samples", tot)
print("stall totals:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v > 0.005 * tot))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for r in sorted(data, key=lambda r: -float(r[ci] or 0))[:n]:
    s = float(r[ci] or 0)
    top = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {r[0]:>6s} {r[si][:70]:70s} " + " ".join(f"{n[6:]}:{v:.0f}" for v, n in top if v > 0))
