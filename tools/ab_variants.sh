#!/bin/bash
# interleaved cfg2 bench A/B of in-tree libhydro variants (base = libhydro.so): bash tools/ab_variants.sh base v1 v2 ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "${BENCH_ARGS[@]}" > gpurun_out/abv_$v.json 2> gpurun_out/abv_$v.err
  python -c "import json;d=json.load(open('gpurun_out/abv_$v.json'));print('$v',round(d['value']/1e6,1),'M k4_ms',round(d['roofline']['k4_ms_per_step'],3))" 2>/dev/null || (echo "$v failed"; tail -3 gpurun_out/abv_$v.err)
done
done
