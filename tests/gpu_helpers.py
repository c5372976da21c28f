"""Shared helpers for the -m gpu parity tests (CUDA path through the C ABI vs oracle/)."""
import numpy as np
import torch

import oracle as O
from paper_2403_14902_b200 import build as B
from paper_2403_14902_b200.hydro import Eddy


def ensure_built():
    B.build()


def make_eddy(w, frames_dev=None, *, policy=None, cost_source="measured", warmup=None, max_batch=None,
              gamma=0.5, max_inflight=4, balance="round_robin"):
    e = Eddy(frames=frames_dev, policy=policy or w.policy, cost_source=cost_source, balance=balance,
             warmup_tuples=w.warmup_tuples if warmup is None else warmup,
             max_batch_tuples=max_batch or w.batch_tuples, decay_gamma=gamma, max_inflight=max_inflight)
    for p in w.preds:
        e.add_predicate(p)
    return e


def run_stream(e, tuples_dev, batch):
    """Submits tuples in routing batches of `batch`, collects in order; returns ids, bboxes, infos."""
    n = len(tuples_dev)
    ids, bbs, infos = [], [], []
    pending = []
    for a in range(0, max(n, 1), batch):
        b = min(a + batch, n)
        pending.append(e.submit(tuples_dev.slice(a, b)))
        if len(pending) >= 2:
            bid = pending.pop(0)
            infos.append(e.batch_info(bid))
            i, bb = e.collect(bid)
            ids.append(i)
            bbs.append(bb)
    for bid in pending:
        infos.append(e.batch_info(bid))
        i, bb = e.collect(bid)
        ids.append(i)
        bbs.append(bb)
    ids = torch.cat(ids).numpy().astype(np.uint64) if ids else np.zeros(0, np.uint64)
    bbs = torch.cat(bbs).numpy().astype(np.int64) if bbs else np.zeros((0, 4), np.int64)
    return ids, bbs, infos


def oracle_result(w, tuples_cpu, frames_np):
    V = O.evaluate_all(w.preds, tuples_cpu, frames_np)
    ids, bbox, keep = O.query_result(tuples_cpu, V)
    return V, ids, bbox, keep


def expected_batch_counters(V, order, warm):
    """Oracle in/pass per predicate for one batch: warmup slice unconditional + chain on the rest."""
    P = V.shape[0]
    n_in = np.zeros(P, np.int64)
    n_pass = np.zeros(P, np.int64)
    if warm > 0:
        n_in += warm
        n_pass += V[:, :warm].sum(1)
    if V.shape[1] > warm:
        a, b, _ = O.sequential_eval(V[:, warm:], order)
        n_in += a
        n_pass += b
    return n_in, n_pass
