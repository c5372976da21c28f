#!/bin/bash
# cfg4 bench (round-robin vs data-aware AREA tiles) per library variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib timeout 900 python bench.py --workload area --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/area_$v.json 2> gpurun_out/area_$v.err
  python -c "import json;d=json.load(open('gpurun_out/area_$v.json'));print('$v', round(d['value']/1e6,1), {k:round(v['ms_per_step'],1) for k,v in d['modes'].items()})" || tail -3 gpurun_out/area_$v.err
done
