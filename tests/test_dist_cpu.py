"""N > 1 host logic on CPU: world size 2 over gloo (127.0.0.1).

Each rank takes its contiguous shard (paper_2403_14902_b200.dist), evaluates it with the oracle under
the current order and follows libhydro's exchange schedule (hydro.h sync_every: every sync_every
batches the window of deltas is all-reduced -- here over gloo, as libhydro's HOST transport does --
and the window of the previous sync point is folded), and must (a) hold the same order as the other
rank at every batch, (b) match the single-process replay of the schedule over both shards
(tests/eddy_replay.py) batch for batch, and (c) together with the other rank reproduce the
1-process result rows in input order.  The same schedule runs inside libhydro with two contexts in
tests/test_gpu_parity.py::test_two_rank_libhydro_host_transport.
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
STEPS = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sync_every, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = workload("cfg2", small=True)
        frames = w.frames().numpy()
        uid = broadcast_unique_id(dist, rank, lambda: bytes(range(128)))
        P = len(w.preds)
        fold = O.FoldState(P, 0.5, [p["declared_cost"] for p in w.preds], cost_source="declared")
        orders, ids = [], []
        window, since, outstanding = np.zeros(2 * P, np.int64), 0, None
        for s in range(STEPS):
            a, b = shard_ids(N_PER_RANK, rank, world, s)
            t = w.tuples(id_start=a, n=b - a)
            V = O.evaluate_all(w.preds, t, frames)
            order = fold.order("score")
            n_in, n_pass, keep = O.sequential_eval(V, order)
            window += np.concatenate([n_in, n_pass])
            since += 1
            if since == sync_every:  # snapshot + exchange this window, fold the previous one
                d = np.array(sum_over_ranks(window.tolist(), dist), np.int64)
                window[:] = 0
                since = 0
                if outstanding is not None:
                    fold.fold(outstanding[:P], outstanding[P:], [0] * P)
                outstanding = d
            orders.append(order)
            ids.append(t.id.numpy()[keep])
        # flush: fold the outstanding window, then exchange and fold the rest
        if outstanding is not None:
            fold.fold(outstanding[:P], outstanding[P:], [0] * P)
        d = np.array(sum_over_ranks(window.tolist(), dist), np.int64)
        fold.fold(d[:P], d[P:], [0] * P)
        gathered = [None] * world
        dist.all_gather_object(gathered, [x.tolist() for x in ids])
        tmax = max_over_ranks(float(rank + 1), dist)
        out[rank] = dict(uid=uid, orders=orders, sel=fold.sel(), rows=gathered, tmax=tmax)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sync_every", [1, 2])
def test_two_rank_shards_merge_to_the_single_process_result(sync_every):
    from tests.eddy_replay import replay

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, sync_every, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["uid"] == r1["uid"] == bytes(range(128))
    assert r0["orders"] == r1["orders"] and r0["sel"] == r1["sel"]
    assert r0["tmax"] == r1["tmax"] == 2.0
    # single process over the same ids: the schedule's replay, and the rows in global order
    w = workload("cfg2", small=True)
    frames = w.frames().numpy()
    Vr = [[], []]
    rows = []
    for s in range(STEPS):
        for r in range(world):
            a, b = shard_ids(N_PER_RANK, r, world, s)
            Vr[r].append(O.evaluate_all(w.preds, w.tuples(id_start=a, n=b - a), frames))
        a, _ = shard_ids(N_PER_RANK, 0, world, s)
        _, b = shard_ids(N_PER_RANK, world - 1, world, s)
        t = w.tuples(id_start=a, n=b - a)
        _, _, keep = O.query_result(t, O.evaluate_all(w.preds, t, frames))
        rows.append(t.id.numpy()[keep])
    rep = replay([np.concatenate(v, axis=1) for v in Vr], N_PER_RANK, 0, [p["declared_cost"] for p in w.preds],
                 sync_every=sync_every, exchange=True)
    assert rep["orders"] == r0["orders"]
    assert rep["fold"].sel() == pytest.approx(r0["sel"], rel=1e-12)
    merged = [i for s in range(STEPS) for r in range(world) for i in r0["rows"][r][s]]
    assert merged == np.concatenate(rows).tolist()


def test_shard_helpers_partition():
    for world in (1, 2, 3, 8):
        spans = [split_range(1001, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 1001
        assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
        ws = [shard_ids(10, r, world, s) for s in range(3) for r in range(world)]
        assert all(ws[i][1] == ws[i + 1][0] for i in range(len(ws) - 1)) and ws[0][0] == 0
