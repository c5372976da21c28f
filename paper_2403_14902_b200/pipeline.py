"""Concurrent workers with cost-driven routing (R29).

The paper routes a batch to the predicate with the lowest *cost* (not the lowest
cost/(1-selectivity) score) when "workers associated with these predicates can run concurrently"
(PAPER.md:327-330): the cheaper stage first keeps the expensive stage -- the bottleneck of the
pipeline -- fed with fewer tuples per unit of time.

On one B200 the workers are hydro contexts, one per predicate, each on its own SM partition (a CUDA
green context: ``sm_groups`` / ``sm_group``) with its own stream, so their kernels run side by side on
disjoint SMs.  A
routing batch visits the workers in the order the policy picks; worker ``order[i+1]`` reads the
survivors of worker ``order[i]`` straight from device memory (``hydro_batch_output`` -> a selection
batch), its stream waiting on the producer batch's done event, so batch b+1's first stage overlaps
batch b's later stages.  Every step runs in libhydro's kernels; this module only sequences the
calls and decides the order (the paper's router), from statistics measured in a warmup phase in
which every worker evaluates the same batch.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Optional, Sequence

import torch

from .hydro import Eddy, hydro_collect_results

POLICIES = ("cost", "score", "selectivity")


def order_by_policy(policy: str, cost: Sequence[float], sel: Sequence[float]) -> List[int]:
    """Lowest key first, ties by predicate id (R2): cost, cost/(1-sel) (PAPER.md:324,
    R1 for s >= 1 / c = 0), selectivity."""
    def key(k):
        c, s = cost[k], sel[k]
        if policy == "cost":
            return c
        if policy == "selectivity":
            return s
        if c == 0.0:
            return 0.0
        return float("inf") if s >= 1.0 else c / (1.0 - s)

    return sorted(range(len(cost)), key=lambda k: (key(k), k))


class ConcurrentEddy:
    """One worker (hydro context + stream + SM budget) per predicate; batches flow through the
    workers in the policy's order, consecutive batches overlapping on different workers."""

    def __init__(self, preds: Sequence[Dict], *, frames: Optional[torch.Tensor] = None, policy: str = "cost",
                 max_batch_tuples: int = 1 << 20, sms: Optional[Sequence[int]] = None, depth: int = 3,
                 partition: str = "green"):
        if policy not in POLICIES:
            raise ValueError(f"policy must be one of {POLICIES}")
        n_sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        P = len(preds)
        sms = list(sms) if sms is not None else [n_sms // P] * P
        self.policy = policy
        self.preds = list(preds)
        self.max_batch = max_batch_tuples
        self.depth = depth
        self.streams = [torch.cuda.Stream() for _ in range(P)]
        self.workers = []
        for k, p in enumerate(preds):
            # "green": worker k owns SM group k of an even split (CUDA green contexts: disjoint SMs);
            # "grid": the grids are only capped at the budget (the CTAs may land on any SM)
            green = partition == "green"
            e = Eddy(frames=frames, policy="fixed", cost_source="measured", warmup_tuples=0,
                     max_batch_tuples=max_batch_tuples, max_inflight=depth + 2, stream=self.streams[k],
                     max_sms=0 if green else int(sms[k]), sm_groups=P if green else 0, sm_group=k if green else 0)
            e.add_predicate(p)
            self.workers.append(e)
        self.sms = sms
        self.order: List[int] = list(range(P))
        self.cost_per_tuple = [1.0] * P   # SM-cycles per tuple (R6) / SMs of the worker
        self.selectivity = [0.5] * P

    # ---- warmup: every worker evaluates the same batch; unconditional statistics
    def warmup(self, tuples) -> List[int]:
        bids = [w.submit(tuples) for w in self.workers]
        for w, b in zip(self.workers, bids):
            w.collect(b)
        for k, w in enumerate(self.workers):
            st = w.stats(0)
            # a worker's time per tuple: its cycles per tuple spread over its SM budget
            self.cost_per_tuple[k] = st["cost_per_tuple"] / max(self.sms[k], 1)
            self.selectivity[k] = st["selectivity"]
        self.order = order_by_policy(self.policy, self.cost_per_tuple, self.selectivity)
        return self.order

    # ---- streaming: batch b's stage i on worker order[i] after stage i-1 (device-side chaining)
    def _submit(self, tuples) -> List[int]:
        chain = []
        for i, k in enumerate(self.order):
            if i == 0:
                chain.append(self.workers[k].submit(tuples))
            else:
                prev = self.order[i - 1]
                pos, cnt, ev = self.workers[prev].batch_output(chain[-1])
                chain.append(self.workers[k].submit(tuples, sel=(pos, cnt, len(tuples)), wait_event=ev))
        return chain

    def _finish(self, chain: List[int], ids_out=None, bb_out=None):
        last = self.workers[self.order[-1]]
        if ids_out is None:
            ids, bb = last.collect(chain[-1])
        else:  # device outputs (bench): no host copy
            n = hydro_collect_results(last.ctx, chain[-1], ids_out.data_ptr(), bb_out.data_ptr(), ids_out.shape[0], 1)
            ids, bb = n, None
        for i in range(len(chain) - 1):  # the earlier stages' survivors were consumed on the device
            self.workers[self.order[i]].release(chain[i])
        return ids, bb

    def run(self, batches, ids_out=None, bb_out=None):
        """Streams the batches through the workers; returns the rows per batch (input order)."""
        pend, out = deque(), []
        for t in batches:
            pend.append(self._submit(t))
            if len(pend) >= self.depth:
                out.append(self._finish(pend.popleft(), ids_out, bb_out))
        while pend:
            out.append(self._finish(pend.popleft(), ids_out, bb_out))
        return out

    def close(self):
        for w in self.workers:
            w.close()
        self.workers = []
