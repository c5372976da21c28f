#!/bin/bash
# K4-T converter warps A/B: parity tests on the variant library, then cfg2 bench lines of both
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
V=$PWD/paper_2403_14902_b200/libhydro_tm16.so
[ -z "$SKIP_TESTS" ] && HYDRO_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
  -k "linear_crops or fused or wide_crops or cfg2 or forced_order or area_and_nearest or cache" > gpurun_out/tm16_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/tm16_tests.log
for rep in 1 2; do
  for v in base tm16; do
    if [ "$v" = "base" ]; then lib=$PWD/paper_2403_14902_b200/libhydro.so; else lib=$V; fi
    HYDRO_LIB_PATH=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg2_$v.json 2> gpurun_out/cfg2_$v.err
    python -c "import json;d=json.load(open('gpurun_out/cfg2_$v.json'));print('$v', round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), round(d['roofline']['k4_ms_per_step'],3))" || tail -3 gpurun_out/cfg2_$v.err
  done
done
