#!/bin/bash
# fused linear pair (K4-T evaluates both heads in one contraction) vs separate hops
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pair_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pair_tests.log
for rep in 1 2; do
for v in pair nopair; do
  if [ $v = nopair ]; then export HYDRO_NO_PAIR=1; else unset HYDRO_NO_PAIR; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abp_$v.json 2> gpurun_out/abp_$v.err
  python -c "import json;d=json.load(open('gpurun_out/abp_$v.json'));print('$v',round(d['value']/1e6,1),'M e2e',round(d['e2e']['value']/1e6,1),'k4_ms',round(d['roofline']['k4_ms_per_step'],3), d['config']['final_order'], d['config']['cost_sm_cycles_per_tuple'])" || tail -5 gpurun_out/abp_$v.err
done
done
