#!/bin/bash
# ncu capture of the K4 AREA hop (legacy SMEM-A kernel) on the cfg4 area bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"hydro_classifier_kernel" -s 6 -c 4 -o gpurun_out/area_full -f \
  python bench.py --workload area --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/area_ncu.log 2>&1
ls -la gpurun_out/area_full.ncu-rep
