#!/bin/bash
# AREA converter check: AREA parity tests, the AREA hop alone per library variant (args), cfg4 bench
# of the base build, ncu of the base build's AREA hop
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "area or cfg4 or data_aware" > gpurun_out/area_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/area_tests.log
bash tools/ab_area2.sh "$@"
timeout 900 python bench.py --workload area --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/area_bench.json 2> gpurun_out/area_bench.err
python -c "import json;d=json.load(open('gpurun_out/area_bench.json'));print('cfg4', round(d['value']/1e6,1), {k:round(v['ms_per_step'],1) for k,v in d['modes'].items()})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hydro_classifier_kernel -s 2 -c 1 -o gpurun_out/area_base -f python tools/area_probe.py 1 > gpurun_out/ncu_base.log 2>&1
