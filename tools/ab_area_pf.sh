#!/bin/bash
# AREA hop A/B over library variants: time (tools/area_probe.py) and ncu DRAM bytes of one launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  echo "$v $(HYDRO_LIB_PATH=$PWD/$lib timeout 300 python tools/area_probe.py 5 2> gpurun_out/probe_$v.err)"
  HYDRO_LIB_PATH=$PWD/$lib timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none \
    -k regex:hydro_classifier_kernel -s 2 -c 1 --csv python tools/area_probe.py 1 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
