cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/l2lim.txt 2>&1
import torch, ctypes
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
from cuda.bindings import runtime as cr
print("default L2 fetch granularity", cr.cudaDeviceGetLimit(cr.cudaLimit.cudaLimitMaxL2FetchGranularity))
PY
for v in none 32 64 128 none 32; do
  if [ $v = none ]; then unset HYDRO_L2_FETCH; else export HYDRO_L2_FETCH=$v; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/l2_$v.json 2>gpurun_out/l2_$v.err
  python -c "import json;d=json.load(open('gpurun_out/l2_$v.json'));print('$v',d['value']/1e6,d['roofline']['k4_ms_per_step'])"
done
export HYDRO_L2_FETCH=32
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hydro_classifier --csv --log-file gpurun_out/l2_32_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/l2_32_launches.csv hydro_classifier_kernel | head -8
cat gpurun_out/l2lim.txt
