#!/bin/bash
# K4-T pair hop under ncu (metrics only) for grid vs general bf16 heads
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for wt in grid bf16; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:hydro_classifier_tm -s 6 -c 1 --csv --log-file gpurun_out/k4t_$wt.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --weights $wt > /dev/null 2>&1
  python - "$wt" <<'PY'
import csv, sys
wt = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/k4t_{wt}.csv")) if len(r) > 5]
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    print(wt, d["Metric Name"], d["Metric Unit"], d["Metric Value"])
PY
done
