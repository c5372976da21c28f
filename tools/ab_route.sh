#!/bin/bash
# A/B the route kernel (R-route evidence run) across in-tree libhydro variants.
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib python bench.py --workload rroute --steps 5 --warmup 3 > gpurun_out/abr_$v.json 2> gpurun_out/abr_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/abr_{v}.json"))
    r = d["roofline"]
    print(f"{v:12s} value={d['value']/1e9:6.2f}G tuples/s  k1_ms/step={r['k1_ms_per_step']:.3f} k2_ms/step={r['k2_ms_per_step']:.3f}  achieved={r['achieved']:.0f} GB/s frac={r['frac']:.3f}")
except Exception as e:
    print(v, "failed", e)
PY
done
