#!/bin/bash
# Bench lines + stamped ncu traffic for the cfg2 headline (grid and bf16 weights).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg2_grid.json 2> gpurun_out/bench_cfg2_grid.err
python bench.py --steps 20 --warmup 5 --weights bf16 --no-cpu-baseline > gpurun_out/bench_cfg2_bf16.json 2> gpurun_out/bench_cfg2_bf16.err
for wt in grid bf16; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hydro \
    --csv --log-file gpurun_out/launches_cfg2_$wt.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --weights $wt > /dev/null 2>&1
  python tools/traffic_json.py gpurun_out/launches_cfg2_$wt.csv hydro_classifier_tm_kernel > gpurun_out/k4_dram_traffic_$wt.json
done
ls -la gpurun_out | tail -12
