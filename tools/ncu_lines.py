"""Stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname = None
out = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            out.append((float(r[4] or 0), fname, r[0], r[1], float(r[7] or 0)))
        except ValueError:
            pass
tot = sum(o[0] for o in out)
for s, f, ln, src, ex in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} inst={ex / 1e6:7.1f}M  {src.strip()[:90]}")
