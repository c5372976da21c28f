"""N > 1 host logic on CPU: world size 2 over gloo (127.0.0.1).

Each rank takes its contiguous shard (paper_2403_14902_b200.dist), evaluates it with the oracle under
a common order, all-reduces the per-predicate deltas exactly like libhydro's ncclAllReduce of the
pending statistics, folds them, and must (a) hold the same order as the other rank, (b) hold the
statistics of a single-process run over all shards, and (c) together with the other rank reproduce
the 1-process result rows in input order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2403_14902_b200.dist import broadcast_unique_id, max_over_ranks, shard_ids, split_range, sum_over_ranks
from synth import workload

N_PER_RANK = 3000
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = workload("cfg2", small=True)
        frames = w.frames().numpy()
        uid = broadcast_unique_id(dist, rank, lambda: bytes(range(128)))
        fold = O.FoldState(len(w.preds), 0.5, [p["declared_cost"] for p in w.preds], cost_source="declared")
        orders, ids = [], []
        for s in range(STEPS):
            a, b = shard_ids(N_PER_RANK, rank, world, s)
            t = w.tuples(id_start=a, n=b - a)
            V = O.evaluate_all(w.preds, t, frames)
            order = fold.order("score")
            n_in, n_pass, keep = O.sequential_eval(V, order)
            d = sum_over_ranks(list(n_in) + list(n_pass), dist)
            P = len(w.preds)
            fold.fold(d[:P], d[P:], [0] * P)
            orders.append(order)
            ids.append(t.id.numpy()[keep])
        gathered = [None] * world
        dist.all_gather_object(gathered, [x.tolist() for x in ids])
        tmax = max_over_ranks(float(rank + 1), dist)
        out[rank] = dict(uid=uid, orders=orders, sel=fold.sel(), rows=gathered, tmax=tmax)
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_merge_to_the_single_process_result():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["uid"] == r1["uid"] == bytes(range(128))
    assert r0["orders"] == r1["orders"] and r0["sel"] == r1["sel"]
    assert r0["tmax"] == r1["tmax"] == 2.0
    # single process over the same ids, in global order
    w = workload("cfg2", small=True)
    frames = w.frames().numpy()
    fold = O.FoldState(len(w.preds), 0.5, [p["declared_cost"] for p in w.preds], cost_source="declared")
    rows = []
    for s in range(STEPS):
        a, _ = shard_ids(N_PER_RANK, 0, world, s)
        _, b = shard_ids(N_PER_RANK, world - 1, world, s)
        t = w.tuples(id_start=a, n=b - a)
        V = O.evaluate_all(w.preds, t, frames)
        order = fold.order("score")
        assert order == r0["orders"][s]
        n_in, n_pass, keep = O.sequential_eval(V, order)
        fold.fold(n_in, n_pass, [0] * len(w.preds))
        rows.append(t.id.numpy()[keep])
    assert fold.sel() == pytest.approx(r0["sel"], rel=1e-12)
    merged = [i for s in range(STEPS) for r in range(world) for i in r0["rows"][r][s]]
    assert merged == np.concatenate(rows).tolist()


def test_shard_helpers_partition():
    for world in (1, 2, 3, 8):
        spans = [split_range(1001, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1001
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        ws = [shard_ids(10, r, world, s) for s in range(3) for r in range(world)]
        assert all(ws[i][1] == ws[i + 1][0] for i in range(len(ws) - 1)) and ws[0][0] == 0
