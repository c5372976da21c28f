"""GPU parity: verdict caches on CLASSIFIER hops (reuse-aware routing on the expensive UDFs,
PAPER.md:589-605, §4.3 UC2; R26).  K0c splits a cached hop into cached verdicts and the
uncached tuples; only those reach the classifier kernel.  Against the oracle's verdicts (the
small workloads' margin-safe caches written by tests/oracle_cache.py): result rows exact, every
per-batch in / pass counter exact (caching never changes which tuples pass), and the evaluated
count of each predicate = its routed tuples minus the cached ones."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import workload
from tests.gpu_helpers import ensure_built, expected_batch_counters, make_eddy, run_stream
from tests.oracle_cache import load

pytestmark = pytest.mark.gpu
N, BATCH = 8000, 2000
CACHED = {1: [(1000, 5000)], 2: [(3000, 7000)]}  # open id intervals per classifier predicate


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ensure_built()


def _setup(name):
    w = workload(name, small=True)
    meta, _, V = load(w.key)
    V = V[:, :N]
    t = w.tuples(n=N)
    keep = V.all(axis=0)
    tid = t.id.numpy().astype(np.int64)
    ref_ids = tid[keep].astype(np.uint64)
    ref_bbox = t.bbox.numpy().astype(np.int64)[keep]
    return w, t, V, tid, ref_ids, ref_bbox


def _cached_mask(ids, k):
    m = np.zeros(len(ids), dtype=bool)
    for lo, hi in CACHED.get(k, []):
        m |= (ids > lo) & (ids < hi)
    return m


def _put(e, tid, V):
    for k in CACHED:
        m = _cached_mask(tid, k)
        e.cache_put(k, torch.from_numpy(tid[m]), torch.from_numpy(V[k][m].astype(np.uint8)))


def _check(ids, bbs, infos, ref_ids, ref_bbox, V, tid, orders=None):
    assert np.array_equal(ids, ref_ids) and np.array_equal(bbs, ref_bbox)
    for b, info in enumerate(infos):
        sl = slice(b * BATCH, (b + 1) * BATCH)
        order = info["order_used"] if orders is None else orders[b]
        assert info["order_used"] == order, (b, info["order_used"], order)
        n_in, n_pass = expected_batch_counters(V[:, sl], order, 0)
        assert info["tuples_in"] == n_in.tolist() and info["tuples_passed"] == n_pass.tolist(), b
        alive = np.ones(BATCH, dtype=bool)
        for k in order:
            want = int((alive & ~_cached_mask(tid[sl], k)).sum())
            assert info["tuples_computed"][k] == want, (b, k, info["tuples_computed"][k], want)
            alive &= V[k, sl]


@pytest.mark.parametrize("name", ["cfg2", "hsv", "mlp"])
def test_classifier_caches_fixed_order(name):
    """Linear (K4-T), HSV and MLP heads with cached verdicts on part of the ids: rows, counters and
    evaluated counts exact under the fixed order label -> breed -> colour."""
    w, t, V, tid, ref_ids, ref_bbox = _setup(name)
    frames = w.frames(device="cuda")
    e = make_eddy(w, frames, policy="fixed", warmup=0, max_batch=BATCH)
    for k in CACHED:
        e.cache_enable(k, 1 << 14)
    _put(e, tid, V)
    ids, bbs, infos = run_stream(e, t.to("cuda"), BATCH)
    e.close()
    _check(ids, bbs, infos, ref_ids, ref_bbox, V, tid, orders=[[0, 1, 2]] * len(infos))


def test_classifier_caches_reuse_policy_orders_by_hit_rate():
    """REUSE policy with declared costs: each batch ordered by (1 - hit) * c from
    its own cache hit rates, exactly as the oracle's reuse_order; rows and counters exact."""
    w, t, V, tid, ref_ids, ref_bbox = _setup("cfg2")
    frames = w.frames(device="cuda")
    e = make_eddy(w, frames, policy="reuse", cost_source="declared", warmup=0, max_batch=BATCH)
    for k in CACHED:
        e.cache_enable(k, 1 << 14)
    _put(e, tid, V)
    ids, bbs, infos = run_stream(e, t.to("cuda"), BATCH)
    e.close()
    costs = [p["declared_cost"] for p in w.preds]
    orders = []
    for b in range(len(infos)):
        bid = tid[b * BATCH:(b + 1) * BATCH]
        hits = [O.cache_hit_rate(bid, CACHED.get(k, [])) for k in range(len(w.preds))]
        orders.append(O.reuse_order(costs, hits))
    assert len({tuple(o) for o in orders}) > 1  # the hit rates change the order across batches
    _check(ids, bbs, infos, ref_ids, ref_bbox, V, tid, orders=orders)


@pytest.mark.parametrize("name", ["cfg2", "hsv"])
def test_classifier_cache_fill_then_reuse(name):
    """fill = 1 records every computed classifier verdict; hydro_cache_fill (UC2's exploratory
    single-UDF query) on the rest; the rerun computes no classifier verdict and
    returns the same rows."""
    w, t, V, tid, ref_ids, ref_bbox = _setup(name)
    frames = w.frames(device="cuda")
    e = make_eddy(w, frames, policy="fixed", warmup=0, max_batch=BATCH)
    for k in CACHED:
        e.cache_enable(k, 1 << 14, fill=True)
    ids, bbs, infos = run_stream(e, t.to("cuda"), BATCH)
    assert np.array_equal(ids, ref_ids) and np.array_equal(bbs, ref_bbox)
    for k in CACHED:  # the tuples a classifier never saw (dropped earlier) through cache_fill
        for a in range(0, N, BATCH):
            e.cache_fill(k, t.slice(a, min(a + BATCH, N)).to("cuda"))
    ids2, bbs2, infos2 = run_stream(e, t.to("cuda"), BATCH)
    e.close()
    assert np.array_equal(ids2, ref_ids) and np.array_equal(bbs2, ref_bbox)
    for info in infos2:
        assert info["tuples_computed"][1] == 0 and info["tuples_computed"][2] == 0, info["tuples_computed"]
