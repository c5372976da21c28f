#!/bin/bash
# compute-sanitizer on the row-cooperative AREA converter (K4, AREA heads) and the data-aware
# warp-level row assignment: memcheck + racecheck over the AREA parity tests
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K="area_crops or wide_and_tall or cfg4_small or data_aware"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "$K" > gpurun_out/memcheck_area.txt 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "area_crops or data_aware_bounds" > gpurun_out/racecheck_area.txt 2>&1
tail -n 5 gpurun_out/memcheck_area.txt gpurun_out/racecheck_area.txt
