#!/bin/bash
# cfg2 bench A/B over library variants (args), interleaved twice on one box
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = "base" ]; then lib=$PWD/paper_2403_14902_b200/libhydro.so; else lib=$PWD/paper_2403_14902_b200/libhydro_$v.so; fi
    HYDRO_LIB_PATH=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg2_$v.json 2> gpurun_out/cfg2_$v.err
    python -c "import json;d=json.load(open('gpurun_out/cfg2_$v.json'));print('$v', round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['k4_ms_per_step'],3))" || tail -3 gpurun_out/cfg2_$v.err
  done
done
