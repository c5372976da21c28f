"""Oracle replay of an eddy run's routing decisions (TEST INFRASTRUCTURE; calls only oracle/).

Given the oracle verdicts of every rank's shard, it replays what the statistics path must do
(SURVEY.md §8(e)): the warmup slice of the first batch on every predicate (R8), one
order per batch from the folded statistics (R4), eager-materialization counters
per batch, and -- with an exchange between ranks -- the window schedule:
every ``sync_every`` batches the window of deltas summed over the ranks is exchanged and the window
exchanged at the PREVIOUS sync point is folded (the warmup slice is exchanged and folded at once;
a final flush folds the rest).  Costs are the declared ones, so the replay is deterministic.
"""
from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np

import oracle as O


def batch_counters(Vb: np.ndarray, order: Sequence[int], warm: int):
    """Oracle in/pass per predicate for one batch: the warmup slice unconditional + the chain on
    the rest (returns the batch totals and the rest-only part)."""
    P = Vb.shape[0]
    w_in = np.zeros(P, np.int64)
    w_pass = np.zeros(P, np.int64)
    if warm > 0:
        w_in += min(warm, Vb.shape[1])
        w_pass += Vb[:, :warm].sum(1)
    r_in = np.zeros(P, np.int64)
    r_pass = np.zeros(P, np.int64)
    if Vb.shape[1] > warm:
        r_in, r_pass, _ = O.sequential_eval(Vb[:, warm:], order)
    return (w_in + r_in, w_pass + r_pass), (r_in, r_pass), (w_in, w_pass)


def replay(V_ranks: List[np.ndarray], batch: int, warm: int, declared: Sequence[float], gamma: float = 0.5,
           sync_every: int = 1, exchange: bool = False, flush: bool = True, policy: str = "score") -> Dict:
    """V_ranks[r] = verdict matrix (P x n_r) of rank r's shard, cut into batches of `batch` (every
    rank the same number of batches).  Returns the expected order of every batch, every rank's
    per-batch counters and the final FoldState."""
    P = V_ranks[0].shape[0]
    nb = max((V.shape[1] + batch - 1) // batch for V in V_ranks)
    fold = O.FoldState(P, gamma, declared, cost_source="declared")
    orders, counters = [], [[] for _ in V_ranks]
    window_in = np.zeros(P, np.int64)
    window_pass = np.zeros(P, np.int64)
    since, outstanding = 0, None
    zero = [0] * P
    if warm > 0:  # the warmup slice: summed over the ranks, folded at once
        d_in = sum(np.full(P, min(warm, V.shape[1]), np.int64) for V in V_ranks)
        d_pass = sum(V[:, :warm].sum(1) for V in V_ranks)
        fold.fold(d_in, d_pass, zero)
    for b in range(nb):
        order = fold.order(policy)
        orders.append(order)
        s_in = np.zeros(P, np.int64)
        s_pass = np.zeros(P, np.int64)
        for r, V in enumerate(V_ranks):
            Vb = V[:, b * batch:(b + 1) * batch]
            tot, rest, _ = batch_counters(Vb, order, warm if b == 0 else 0)
            counters[r].append(tot)
            s_in += rest[0]
            s_pass += rest[1]
        if not exchange:
            fold.fold(s_in, s_pass, zero)
            continue
        window_in += s_in
        window_pass += s_pass
        since += 1
        if since == sync_every:
            snap = (window_in.copy(), window_pass.copy())
            window_in[:] = 0
            window_pass[:] = 0
            since = 0
            if outstanding is not None:
                fold.fold(outstanding[0], outstanding[1], zero)
            outstanding = snap
    if exchange and flush:
        if outstanding is not None:
            fold.fold(outstanding[0], outstanding[1], zero)
        fold.fold(window_in, window_pass, zero)
    return dict(orders=orders, counters=counters, fold=fold)
