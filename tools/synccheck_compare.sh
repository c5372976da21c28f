#!/bin/bash
# synccheck on the K4-T kernel with the default staging wait and with a test_wait spin (tool check)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in base tw; do
  if [ $v = base ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  HYDRO_LIB_PATH=$PWD/$lib timeout 900 compute-sanitizer --tool synccheck --print-limit 3 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "linear_crops" > gpurun_out/synccheck_$v.txt 2>&1
  echo "== $v"; tail -3 gpurun_out/synccheck_$v.txt; grep -m1 -A5 "Barrier error" gpurun_out/synccheck_$v.txt
done
