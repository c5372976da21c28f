"""Diagnostic for the UC2 evidence run: per-batch order and K1 time under each policy."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_14902_b200 import build as B
from paper_2403_14902_b200 import hydro as H
from synth import workload

B.build()
n, batch, scale, units = 15_000_000, 1_000_000, 1000, int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = workload("uc2", n=n)
for p in w.preds:
    p["units"], p["declared_cost"] = units, float(units)
t = w.tuples(device="cuda")
ranges = [(1000 * scale, 7000 * scale), (8000 * scale, 14000 * scale)]
for policy in ("fixed", "reuse"):
    e = H.Eddy(policy=policy, warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4)
    for p in w.preds:
        e.add_predicate(p)
    for k, (lo, hi) in enumerate(ranges):
        e.cache_enable(k, n)
        for a in range(lo + 1, hi, batch):
            e.cache_fill(k, t.slice(a, min(a + batch, hi)))
    if policy == "fixed":
        e.set_fixed_order([0, 1])
    for rep in range(2):
        e.set_kernel_timing(True)
        rows = []
        for a in range(0, n, batch):
            e.set_kernel_timing(True)
            bid = e.submit(t.slice(a, a + batch))
            info = e.batch_info(bid)
            e.collect(bid, device="cuda")
            rows.append((info["order_used"], info["tuples_computed"], round(e.kernel_time(0)[0], 3)))
        k1 = e.kernel_time(0)
        k2 = e.kernel_time(3)
        k5 = e.kernel_time(2)
        e.set_kernel_timing(False)
        if rep == 1:
            print(policy, "K1 ms", round(k1[0], 3), k1[1], "K2", round(k2[0], 3), "K5", round(k5[0], 3))
            for i, r in enumerate(rows):
                print("  batch", i, r)
    e.close()
