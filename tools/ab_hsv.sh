#!/bin/bash
# HSV dog-query bench per library variant (the HSV hop's kernel rate is in the line's roofline)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=$PWD/paper_2403_14902_b200/libhydro.so; else lib=$PWD/paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$lib timeout 600 python bench.py --workload hsv --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hsv_$v.json 2> gpurun_out/hsv_$v.err
  python -c "import json;d=json.load(open('gpurun_out/hsv_$v.json'));r=d['roofline'];print('$v', round(d['value']/1e6,1), round(r['hsv_ms_per_step'],3), round(r['hsv_kernel_tuples_per_s']/1e6,1))" || tail -3 gpurun_out/hsv_$v.err
done
