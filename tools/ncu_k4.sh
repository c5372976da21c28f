#!/bin/bash
# One full ncu capture (source-level) of the K4 breed hop of the cfg2 bench command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=${1:-k4}
shift
ncu --set full --clock-control none --import-source on -k regex:hydro_classifier -s 6 -c 1 -o gpurun_out/${tag}_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${tag}_ncu.log 2>&1
ls -la gpurun_out/${tag}_full.ncu-rep
