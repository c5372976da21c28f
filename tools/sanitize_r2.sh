#!/bin/bash
# Round-2 compute-sanitizer passes: the new kernels (K4-T linear heads with bulk staging and TMEM A,
# K0c classifier cache split + redirected K4 / HSV / MLP, K1F fused route+emit) plus the K4 linear
# and MLP kernels under racecheck / synccheck (round 1 ran those two tools on other kernels only).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K="cfg1 or edge or linear_crops or mlp_crops or hsv_counts or cfg3 or area_crops or mlp_query"
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cache.py -x -q -p no:cacheprovider \
  -k "$K or fixed_order or reuse_policy or fill_then" > gpurun_out/memcheck_r2.txt 2>&1
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cache.py -x -q -p no:cacheprovider \
  -k "cfg1 or linear_crops or mlp_crops or hsv_counts or fixed_order" > gpurun_out/racecheck_r2.txt 2>&1
timeout 2400 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cache.py -x -q -p no:cacheprovider \
  -k "cfg1 or linear_crops or mlp_crops or fixed_order" > gpurun_out/synccheck_r2.txt 2>&1
tail -n 4 gpurun_out/memcheck_r2.txt gpurun_out/racecheck_r2.txt gpurun_out/synccheck_r2.txt
