#!/bin/bash
# One GPU call that produces the round's measurement artefacts under gpurun_out/ (copied to
# profiles/ by hand after review): bench lines (cfg2 with the oracle baseline, R-route), the ncu
# launch list of the cfg2 bench command, one full capture of the K4 breed hop and of K1/K2 on R-route.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --workload rroute --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rroute.json 2> gpurun_out/bench_rroute.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hydro \
  --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:hydro_classifier -s 6 -c 3 -o gpurun_out/k4_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hydro_route|hydro_compact" -s 20 -c 2 -o gpurun_out/route_full -f \
  python bench.py --workload rroute --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -12
