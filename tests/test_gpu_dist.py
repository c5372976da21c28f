"""Multi-rank libhydro on one GPU (a11; "Scaling Out").

gpurun gives one GPU, so N ranks run as N processes on cuda:0, each with its own hydro context, and
the statistics exchange goes through libhydro's HOST transport (a gloo all-reduce callback) -- the
same snapshot -> exchange -> fold-one-sync-late path as the NCCL transport of an N-GPU run.  Checked:
every rank uses the same order at every batch, that order and every per-rank per-batch counter equal
the oracle replay of the schedule (tests/eddy_replay.py), the rank-ordered union of the rows equals
the single-rank rows, which equal the oracle's, and the flushed statistics equal the replay's.
"""
import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
from paper_2403_14902_b200.dist import shard_ids
from synth import workload
from tests.eddy_replay import replay
from tests.gpu_helpers import ensure_built

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ensure_built()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(world, spec):
    from tests.dist_hydro_worker import run

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(run, args=(world, _free_port(), spec, d), nprocs=world, join=True, start_method="spawn")
        out = []
        for r in range(world):
            with open(os.path.join(d, f"rank{r}.pkl"), "rb") as f:
                out.append(pickle.load(f))
    return out


@pytest.mark.parametrize("world,sync_every", [(2, 1), (2, 3), (3, 2)])
def test_two_rank_libhydro_host_transport(world, sync_every):
    spec = dict(workload="cfg2", batch=1200, batches=5, warm=512, sync_every=sync_every)
    res = _run_ranks(world, spec)
    w = workload("cfg2", small=True)
    frames = w.frames().numpy()
    P = len(w.preds)
    # oracle verdicts of every rank's shard (batches in order)
    V_ranks = []
    for r in range(world):
        parts = []
        for s in range(spec["batches"]):
            a, b = shard_ids(spec["batch"], r, world, s)
            parts.append(O.evaluate_all(w.preds, w.tuples(id_start=a, n=b - a), frames))
        V_ranks.append(np.concatenate(parts, axis=1))
    rep = replay(V_ranks, spec["batch"], spec["warm"], [p["declared_cost"] for p in w.preds],
                 sync_every=sync_every, exchange=True)
    for r in range(world):
        got = [i["order_used"] for i in res[r]["infos"]]
        assert got == rep["orders"], (r, got, rep["orders"])
        for s, info in enumerate(res[r]["infos"]):
            n_in, n_pass = rep["counters"][r][s]
            assert info["tuples_in"] == n_in.tolist() and info["tuples_passed"] == n_pass.tolist(), (r, s)
        # flushed statistics: identical on every rank and equal to the replay's fold
        for k in range(P):
            assert res[r]["stats"][k]["selectivity"] == pytest.approx(rep["fold"].sel()[k], rel=1e-12)
            assert res[r]["stats"][k]["s_in"] == res[0]["stats"][k]["s_in"]
        assert res[r]["order"] == res[0]["order"]
    # exchanges: one per sync point + the warmup slice's + the flush's
    assert res[0]["calls"] == spec["batches"] // sync_every + 2
    # rank-ordered union of the rows == the global result in input order == the oracle's
    ids = np.concatenate([res[r]["ids"][s] for s in range(spec["batches"]) for r in range(world)]).astype(np.uint64)
    bbs = np.concatenate([res[r]["bbs"][s] for s in range(spec["batches"]) for r in range(world)]).astype(np.int64)
    n_all = world * spec["batch"] * spec["batches"]
    t = w.tuples(n=n_all)
    V = O.evaluate_all(w.preds, t, frames)
    ref_ids, ref_bb, _ = O.query_result(t, V)
    assert np.array_equal(ids, ref_ids) and np.array_equal(bbs, ref_bb)


def test_host_transport_single_rank_equals_nccl_single_rank():
    """world = 1 with an exchange: the HOST callback path and the 1-rank NCCL communicator path run the
    same schedule (snapshot, exchange, fold one sync late) and give identical orders, counters and
    statistics, equal to the replay."""
    from paper_2403_14902_b200 import hydro as H
    from tests.gpu_helpers import run_stream

    w = workload("cfg2", small=True, n=12000)
    frames = w.frames()
    t = w.tuples().to("cuda")
    runs = []
    for mode in ("host", "nccl"):
        kw = dict(allreduce=lambda x: None) if mode == "host" else dict(nccl_unique_id=H.hydro_nccl_unique_id())
        e = H.Eddy(frames=frames.cuda(), policy="score", cost_source="declared", warmup_tuples=1024,
                   max_batch_tuples=3000, world=1, rank=0, sync_every=2, **kw)
        for p in w.preds:
            e.add_predicate(p)
        ids, bbs, infos = run_stream(e, t, 3000)
        e.flush_stats()
        runs.append((ids, bbs, [i["order_used"] for i in infos], [e.stats(k)["selectivity"] for k in range(3)]))
        e.close()
    (i0, b0, o0, s0), (i1, b1, o1, s1) = runs
    assert np.array_equal(i0, i1) and np.array_equal(b0, b1) and o0 == o1 and s0 == s1
    V = O.evaluate_all(w.preds, w.tuples(), frames.numpy())
    rep = replay([V], 3000, 1024, [p["declared_cost"] for p in w.preds], sync_every=2, exchange=True)
    assert o0 == rep["orders"]
    assert s0 == pytest.approx(rep["fold"].sel(), rel=1e-12)
