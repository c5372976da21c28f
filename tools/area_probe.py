"""AREA hop probe: cfg4's AREA breed head ALONE over 1M cfg4 tuples per batch (every tuple a crop),
device-timed; prints crops/s, the mean source pixels per crop and the algorithmic DRAM rate
(w*h*3 bytes per crop).  Usage: python tools/area_probe.py [steps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_14902_b200 import hydro as H  # noqa: E402
from synth import workload  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = 1 << 20
w = workload("cfg4", n=n)
frames = w.frames(device="cuda")
t = w.tuples(device="cuda")
p = w.preds[3]
assert p["crop_mode"] == "area"
stream = torch.cuda.current_stream()
e = H.Eddy(frames=frames, policy="fixed", warmup_tuples=0, max_batch_tuples=n, stream=stream)
e.add_predicate(p)
res_ids = torch.empty(n, dtype=torch.int64, device="cuda")
res_bb = torch.empty((n, 4), dtype=torch.int16, device="cuda")
for _ in range(2):
    e.collect_into(e.submit(t), res_ids, res_bb)
torch.cuda.synchronize()
ms = []
for _ in range(steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    e.collect_into(e.submit(t), res_ids, res_bb)
    b.record(stream)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
e.close()
bb = t.bbox.long().cpu()
area = ((bb[:, 2] - bb[:, 0]) * (bb[:, 3] - bb[:, 1])).double()
m = sorted(ms)[len(ms) // 2]
print(json.dumps({"crops": n, "ms": m, "crops_per_s": n / m * 1e3, "mean_px": area.mean().item(),
                  "alg_gbs": float(area.sum() * 3 / (m * 1e-3) / 1e9)}))
