#!/bin/bash
# A/B the in-tree libhydro variants on the R-route evidence run (K1/K2).
# usage (under gpurun): bash tools/ab_route.sh base prev ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib python bench.py --workload rroute --steps 5 --warmup 3 > gpurun_out/abr_$v.json 2> gpurun_out/abr_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/abr_{v}.json"))
    r, l = d["roofline"], d["roofline_label_only"]
    print(f"{v:8s} chain={d['value']/1e9:6.1f}G frac={r['frac']:.3f} k1={r['k1_ms_per_step']:.3f} k2={r['k2_ms_per_step']:.3f} | "
          f"label-only frac={l['frac']:.3f} k1={l['k1_ms_per_step']:.3f} k2={l['k2_ms_per_step']:.3f}")
except Exception as e:
    print(v, "failed", e)
PY
done
