#!/bin/bash
# AREA converter A/B (cfg4 area bench) after the AREA parity tests: base vs prev
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -m gpu -x -q -p no:cacheprovider -k "area or cfg4 or data_aware or balance" > gpurun_out/area_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/area_tests.log
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib timeout 900 python bench.py --workload area --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/area_$v.json 2> gpurun_out/area_$v.err
  python -c "import json;d=json.load(open('gpurun_out/area_$v.json'));print('$v', round(d['value']/1e6,1), {k:round(v['ms_per_step'],1) for k,v in d['modes'].items()})" || tail -3 gpurun_out/area_$v.err
done
