#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/k1f_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/k1f_tests.log
for v in fused legacy fused legacy; do
  if [ $v = legacy ]; then export HYDRO_NO_K1F=1; else unset HYDRO_NO_K1F; fi
  python bench.py --workload small --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/small_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/small_$v.json'));print('$v', d['cfg1']['us_per_batch_device'], d['cfg1']['us_per_batch_host'], {k:round(d['cfg3'][k]['tuples_per_s']/1e6,1) for k in ('score','static')})"
done
unset HYDRO_NO_K1F
python bench.py --workload rroute --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/rr.json 2>gpurun_out/rr.err; head -c 400 gpurun_out/rr.json
