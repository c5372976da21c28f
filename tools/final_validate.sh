#!/bin/bash
# End-of-round GPU run: every -m gpu test and smoke, then the round-2 profile artefacts
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
tail -2 gpurun_out/final_gputest.log; tail -2 gpurun_out/final_smoke.log
bash tools/round2_profiles.sh
