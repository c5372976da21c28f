#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/tm_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/tm_parity.log
bash tools/ab_variants.sh "$@"
