"""ncu helper: the label-only chain (routing + compaction, no UDF arithmetic) on 16M-tuple batches."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2403_14902_b200 import hydro as H  # noqa: E402
from synth import label_pred, workload  # noqa: E402

batch = 1 << 24
w = workload("cfg2", n=batch)
t = [w.tuples(id_start=b * batch, n=batch, device="cuda") for b in range(2)]
e = H.Eddy(policy="score", warmup_tuples=65536, max_batch_tuples=batch, stream=torch.cuda.current_stream())
e.add_predicate(label_pred())
res_ids = torch.empty(batch, dtype=torch.int64, device="cuda")
res_bb = torch.empty((batch, 4), dtype=torch.int16, device="cuda")
for s in range(6):
    bid = e.submit(t[s % 2])
    H.hydro_collect_results(e.ctx, bid, res_ids.data_ptr(), res_bb.data_ptr(), batch, 1)
torch.cuda.synchronize()
e.close()
