#!/bin/bash
# A/B the in-tree libhydro variants on the R-route workload (K1/K2 evidence run).
# usage (under gpurun): bash tools/ab_route.sh base old ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib python bench.py --workload rroute --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abr_$v.json 2> gpurun_out/abr_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/abr_{v}.json"))
    r = d["roofline"]
    print(f"{v:8s} value={d['value']/1e9:6.1f}G  frac={r['frac']:.3f} step_frac={r.get('frac_over_step', 0):.3f} k1={r['k1_ms_per_step']:.3f} k2={r['k2_ms_per_step']:.3f} label_only={d['roofline_label_only']['frac']:.3f}")
except Exception as e:
    print(v, "failed", e, open(f"gpurun_out/abr_{v}.err").read()[-500:])
PY
done
