#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for wl in cfg2 mlp hsv; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/qb_$wl.json 2> gpurun_out/qb_$wl.err
  python -c "import json;d=json.load(open('gpurun_out/qb_$wl.json'));r=d['roofline'];print('$wl',round(d['value']/1e6,1),'M frac',round(r['frac'],3),'items/step',r.get('classifier_tuples_per_step'),r.get('head_evaluations_per_step'))" || tail -3 gpurun_out/qb_$wl.err
done
