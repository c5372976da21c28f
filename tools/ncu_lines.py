"""Stall samples and executed warp instructions per CUDA source line from
`ncu -i rep --page source --csv --print-source cuda,sass` (metrics counted from the end of a row,
so source text containing commas does not shift them).
    python tools/ncu_lines.py src.csv [top] [file:lo-hi ...]   # ranges: summed instruction counts"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
nm = len(hdr) - 2  # Address, Source (SASS), then the metrics
fname = None
out = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) >= len(hdr) and r[0].isdigit():
        m = r[len(r) - nm:]
        try:
            out.append((float(m[2] or 0), fname, int(r[0]), ",".join(r[1:len(r) - nm]), float(m[5] or 0)))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1.0
itot = sum(o[4] for o in out)
print(f"total warp instructions {itot / 1e9:.2f}G, stall samples {tot:.0f}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, f, ln, src, ex in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} inst={ex / 1e6:8.1f}M  {src.strip()[:90]}")
for spec in sys.argv[3:]:
    f, rng = spec.split(":")
    lo, hi = (int(x) for x in rng.split("-"))
    sel = [o for o in out if o[1] == f and lo <= o[2] <= hi]
    print(f"{spec}: inst {sum(o[4] for o in sel) / 1e9:.3f}G, stall {100 * sum(o[0] for o in sel) / tot:.1f}%")
