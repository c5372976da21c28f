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
calls; the order (the paper's router) is decided inside libhydro (``hydro_route_workers``, a device
kernel over the workers' folded statistics) after a warmup phase in which every worker evaluates the
same batch.
"""
from __future__ import annotations

from collections import deque
from typing import Dict, List, Optional, Sequence

import torch

from .hydro import Eddy, hydro_route_workers

POLICIES = ("cost", "score", "selectivity")


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
        self.cost_per_tuple = [1.0] * P   # reported by the router: SM-cycles per tuple (R6) / worker SMs
        self.selectivity = [0.5] * P

    # ---- warmup: every worker evaluates the same batch; unconditional statistics
    @staticmethod
    def _producer_event():
        """Event on the caller's current stream: the workers' first kernels wait for the work that
        produced the tuples (the workers run on their own streams)."""
        ev = torch.cuda.Event()
        ev.record()
        return ev

    def warmup(self, tuples) -> List[int]:
        ev = self._producer_event()
        bids = [w.submit(tuples, wait_event=ev.cuda_event) for w in self.workers]
        for w, b in zip(self.workers, bids):
            w.collect(b)
        self.order, self.cost_per_tuple, self.selectivity = hydro_route_workers([w.ctx for w in self.workers],
                                                                                self.policy)
        return self.order

    # ---- streaming: batch b's stage i on worker order[i] after stage i-1 (device-side chaining)
    def _submit(self, tuples) -> List[int]:
        chain = []
        ev = self._producer_event()
        for i, k in enumerate(self.order):
            if i == 0:
                chain.append(self.workers[k].submit(tuples, wait_event=ev.cuda_event))
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
            n = last.collect_into(chain[-1], ids_out, bb_out)
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
