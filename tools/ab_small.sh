#!/bin/bash
# latency / adaptation configs (bench --workload small) per library variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=$PWD/paper_2403_14902_b200/libhydro.so; else lib=$PWD/paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$lib timeout 600 python bench.py --workload small > gpurun_out/small_$v.json 2> gpurun_out/small_$v.err
  python -c "import json;d=json.load(open('gpurun_out/small_$v.json'));c=d['cfg3'];print('$v', 'cfg1 us', round(d['cfg1']['us_per_batch_host'],1), round(d['cfg1']['us_per_batch_device'],1), 'cfg3', {k:(round(v['tuples_per_s']/1e6,1) if isinstance(v,dict) and 'tuples_per_s' in v else None) for k,v in c.items() if isinstance(v,dict)})" || tail -3 gpurun_out/small_$v.err
done
