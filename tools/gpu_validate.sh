#!/bin/bash
# One-call GPU validation: gpu tests, smoke, cfg2 bench lines (grid + bf16 weights), the
# launch list of the bench command and the stamped K4 DRAM traffic.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
bash tools/gpu_bench_round2.sh
tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log
cat gpurun_out/bench_cfg2_grid.json gpurun_out/bench_cfg2_bf16.json
