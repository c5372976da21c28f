"""Top stall-sampled SASS instructions of an ncu source page export (--page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data)
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
print("total samples", tot)
for d in sorted(data, key=lambda d: -float(d[key] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    s = float(d[key] or 0)
    top = sorted(((float(d[c] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{d['Address']:>6} {100*s/tot:5.1f}% {d['Source'][:70]:70s} " + " ".join(f"{c}={v:.0f}" for v, c in top if v))
