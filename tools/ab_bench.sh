#!/bin/bash
# A/B the in-tree libhydro variants on the GPU box: one short bench per variant.
# usage (under gpurun): bash tools/ab_bench.sh base predlds nopf ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{v}.json"))
    print(f"{v:14s} value={d['value']/1e6:7.1f}M  e2e={d['e2e']['value']/1e6:7.1f}M  k4_ms/step={d['roofline']['k4_ms_per_step']:.3f}  frac={d['roofline']['frac']:.3f}  clocks={d['clocks']}")
except Exception as e:
    print(v, "failed", e)
PY
done
