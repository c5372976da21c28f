#!/bin/bash
# Round-2 measurement artefacts (copied to profiles/ after review): bench lines of every workload,
# the ncu launch list of the cfg2 bench command (+ stamped K4-T DRAM traffic), one full ncu capture
# of the K4-T breed hop and of K1/K2 on R-route.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
O=gpurun_out/r2
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --weights bf16 --no-cpu-baseline > $O/bench_cfg2_bf16.json 2> $O/bench_cfg2_bf16.err
for wl in rroute mlp hsv uc2 uc2cls area small concurrent orders; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hydro \
  --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/traffic_json.py $O/launches_cfg2.csv hydro_classifier_tm_kernel > $O/k4_dram_traffic.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hydro \
  --csv --log-file $O/launches_cfg2_bf16.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --weights bf16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:hydro_classifier_tm -s 6 -c 1 -o $O/k4t_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"hydro_route|hydro_compact" -s 20 -c 2 -o $O/route_full -f \
  python bench.py --workload rroute --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# R-route launch list: DRAM bytes of K1 and K2 per 16M-tuple batch (stamped, bench.py's rroute traffic)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"hydro_route|hydro_compact" \
  --csv --log-file $O/launches_rroute.csv env HYDRO_ROUTE_ONLY=1 python bench.py --workload rroute --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/traffic_json.py $O/launches_rroute.csv hydro_route_kernel > $O/route_k1_dram_traffic.json
python tools/traffic_json.py $O/launches_rroute.csv hydro_compact_kernel > $O/route_k2_dram_traffic.json
# the AREA hop alone (cfg4's AREA head on 1M crops, 16-converter-warp K4 instance)
python tools/area_probe.py 5 > $O/area_probe.json 2> $O/area_probe.err
ncu --set full --clock-control none --import-source on -k regex:hydro_classifier_kernel -s 2 -c 1 -o $O/area_full -f \
  python tools/area_probe.py 1 > /dev/null 2>&1
ls -la $O
