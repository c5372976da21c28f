#!/bin/bash
# compute-sanitizer passes over a subset of the GPU parity tests (one GPU; under gpurun).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "cfg1 or edge or uc2_reuse or hsv_counts or linear_crops or mlp_crops or (data_aware and 700) or selection_chain or area_crops or route_full or cfg3" \
  > gpurun_out/memcheck.txt 2>&1
compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "cfg1 or uc2_reuse or hsv_counts or edge or (data_aware and 9000)" > gpurun_out/racecheck.txt 2>&1
compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q \
  -k "cfg1 or uc2_reuse or hsv_counts or (data_aware and 9000)" > gpurun_out/synccheck.txt 2>&1
tail -n 3 gpurun_out/memcheck.txt gpurun_out/racecheck.txt gpurun_out/synccheck.txt
