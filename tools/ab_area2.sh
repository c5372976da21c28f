#!/bin/bash
# AREA converter A/B: the AREA hop alone (tools/area_probe.py) per library variant, then cfg4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = "base" ]; then lib=paper_2403_14902_b200/libhydro.so; else lib=paper_2403_14902_b200/libhydro_$v.so; fi
  echo "$v $(HYDRO_LIB_PATH=$PWD/$lib timeout 300 python tools/area_probe.py 5 2> gpurun_out/probe_$v.err)"
done
