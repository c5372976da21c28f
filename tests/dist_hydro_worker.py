"""One rank of a world-size-N libhydro run on ONE GPU (test infrastructure for
tests/test_gpu_dist.py): every rank is its own process with its own hydro context on cuda:0, and the
statistics exchange (a11) goes through libhydro's HOST transport -- a gloo all-reduce called back
from inside hydro_submit_batch / hydro_flush_stats -- through the same PREP -> snapshot -> exchange ->
fold path the NCCL transport takes on N GPUs.
"""
from __future__ import annotations

import os
import pickle

import numpy as np
import torch
import torch.distributed as dist

from paper_2403_14902_b200.dist import shard_ids
from paper_2403_14902_b200.hydro import Eddy
from synth import workload


def run(rank: int, world: int, port: int, spec: dict, out_dir: str):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        w = workload(spec["workload"], small=True)
        frames = w.frames().cuda() if w.needs_frames else None
        calls = []

        def allreduce(t):  # HOST transport: sum over the ranks, in place
            calls.append(int(t.numel()))
            dist.all_reduce(t)

        e = Eddy(frames=frames, policy="score", cost_source="declared", warmup_tuples=spec["warm"],
                 max_batch_tuples=spec["batch"], world=world, rank=rank, sync_every=spec["sync_every"],
                 allreduce=allreduce if world > 1 or spec.get("host_at_world1") else None)
        for p in w.preds:
            e.add_predicate(p)
        infos, ids, bbs = [], [], []
        for s in range(spec["batches"]):
            a, b = shard_ids(spec["batch"], rank, world, s)
            t = w.tuples(id_start=a, n=b - a).to("cuda")
            bid = e.submit(t)
            infos.append(e.batch_info(bid))
            i, bb = e.collect(bid)
            ids.append(i.numpy())
            bbs.append(bb.numpy())
        e.flush_stats()
        stats = [e.stats(k) for k in range(len(w.preds))]
        res = dict(rank=rank, infos=infos, ids=ids, bbs=bbs, stats=stats, order=e.order(), calls=len(calls))
        e.close()
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
    finally:
        dist.destroy_process_group()
