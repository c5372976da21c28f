#!/bin/bash
# K4-T (A in TMEM) vs the shared-memory-A kernel: GPU parity first, then an interleaved bench A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/tm_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/tm_parity.log
tail -5 gpurun_out/tm_parity.log
for v in tm legacy tm legacy; do
  if [ $v = legacy ]; then export HYDRO_K4_LEGACY=1; else unset HYDRO_K4_LEGACY; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abtm_$v.json 2> gpurun_out/abtm_$v.err
  python -c "import json;d=json.load(open('gpurun_out/abtm_$v.json'));print('$v',round(d['value']/1e6,1),'M k4_ms',round(d['roofline']['k4_ms_per_step'],3))" || tail -5 gpurun_out/abtm_$v.err
done
