import torch
from paper_2403_14902_b200.hydro import Eddy
torch.cuda.init()
for g in (0, 1):
    try:
        e = Eddy(policy="fixed", warmup_tuples=0, max_batch_tuples=4096, sm_groups=2, sm_group=g)
        print("group", g, "ok"); e.close()
    except Exception as ex:
        print("group", g, "fail", ex)
