"""Full-set parity at BASELINE.json sizes (SURVEY.md §8(d) "Coverage"): the CUDA path through the C ABI,
in the bench's launch configuration, against the oracle verdicts cached on disk by
tests/oracle_cache.py (which calls only oracle/), compared on EVERY row and EVERY per-batch counter.

  cfg2 (1M dog-query tuples, linear heads)     every row + counters, grid and general-bf16 weights
  cfg4 (10M tuples; its 1M prefix)              every row + counters, data-aware AREA tiles
  cfg5 (100M tuples over 8 shards)              every tuple of the 1 % sample id % 100 == 0
  mlp / hsv (the f1 / f4 dog queries, 1M)       every row + counters

Every classifier margin of the covered tuples is >= 0.05 by construction (the cache's bbox redraw
table, R12), so verdicts are compared without any test-time filtering.
"""
import numpy as np
import pytest
import torch

import oracle as O
from synth import shard_range, workload
from tests.eddy_replay import batch_counters
from tests.gpu_helpers import ensure_built, make_eddy, run_stream
from tests.oracle_cache import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ensure_built()


def _check_run(w, V, ids, bbs, infos, batch, warm, n):
    t = w.tuples(n=n)
    ref_ids, ref_bb, _ = O.query_result(t, V[:, :n])
    assert ids.shape == ref_ids.shape, (ids.shape, ref_ids.shape)
    assert np.array_equal(ids, ref_ids) and np.array_equal(bbs, ref_bb)
    for b, info in enumerate(infos):
        Vb = V[:, b * batch:min((b + 1) * batch, n)]
        (n_in, n_pass), _, _ = batch_counters(Vb, info["order_used"], warm if b == 0 else 0)
        assert info["tuples_in"] == n_in.tolist() and info["tuples_passed"] == n_pass.tolist(), b


@pytest.mark.parametrize("weights", ["grid", "bf16"])
@pytest.mark.parametrize("batch", [1 << 20, 1 << 17])
def test_cfg2_every_row_and_counter(weights, batch):
    """cfg2 at BASELINE size: one 1M-tuple batch (the bench's batch) and 8 batches of 128K (SURVEY.md
    §8(a) a1), score policy with measured costs; every row and every batch's counters exact."""
    w = workload("cfg2", weights=weights)
    meta, _, V = load(w.key)
    assert meta["covered"] == w.n == 1_000_000 and meta["min_abs_margin"][1] >= 0.05
    e = make_eddy(w, w.frames(device="cuda"), policy="score", warmup=65536, max_batch=batch)
    ids, bbs, infos = run_stream(e, w.tuples().to("cuda"), batch)
    e.close()
    _check_run(w, V, ids, bbs, infos, batch, 65536, w.n)


@pytest.mark.parametrize("weights", ["grid", "bf16"])
def test_cfg4_prefix_every_row_and_counter(weights):
    """cfg4 (10M tuples, area-correlated cost) on its first 1M tuples (the oracle's AREA crops make the
    full 10M a multi-hour CPU run), in the area bench's configuration: 1M-tuple batches, data-aware
    tiles for the AREA hop.  Every row and counter exact."""
    w = workload("cfg4", weights=weights)
    meta, _, V = load(w.key)
    n = meta["covered"]
    assert n == 1_000_000
    e = make_eddy(w, w.frames(device="cuda"), policy="score", warmup=65536, max_batch=1 << 18, balance="data_aware")
    ids, bbs, infos = run_stream(e, w.tuples(n=n).to("cuda"), 1 << 18)
    e.close()
    _check_run(w, V, ids, bbs, infos, 1 << 18, 65536, n)


@pytest.mark.parametrize("name", ["mlp", "hsv"])
def test_f1_f4_dog_queries_every_row_and_counter(name):
    w = workload(name)
    meta, _, V = load(w.key)
    assert meta["covered"] == w.n
    e = make_eddy(w, w.frames(device="cuda"), policy="score", warmup=65536, max_batch=1 << 20)
    ids, bbs, infos = run_stream(e, w.tuples().to("cuda"), 1 << 20)
    e.close()
    _check_run(w, V, ids, bbs, infos, 1 << 20, 65536, w.n)


def test_cfg5_eight_shards_one_percent_sample():
    """cfg5: the dog query on 100M tuples sharded contiguously over 8 ranks (each shard through its own
    context, 1M-tuple batches); the rank-ordered union is in input order without duplicates, every
    returned bbox is the tuple's, and membership of EVERY tuple of the 1 % sample equals the oracle's."""
    w = workload("cfg5")
    meta, sample_ids, V = load(w.key)
    assert meta["mode"] == "mod100" and len(sample_ids) == 1_000_000
    frames = w.frames(device="cuda")
    got_sample = []
    last = -1
    for r in range(8):
        a, b = shard_range(w.n, r, 8)
        t = w.tuples(id_start=a, n=b - a, device="cuda")
        e = make_eddy(w, frames, policy="score", warmup=65536, max_batch=1 << 20)
        ids, bbs, _ = run_stream(e, t, 1 << 20)
        e.close()
        ids64 = ids.astype(np.int64)
        assert ids64.min() >= a and ids64.max() < b and ids64[0] > last and np.all(np.diff(ids64) > 0)
        last = int(ids64[-1])
        pos = torch.from_numpy(ids64 - a).cuda()
        assert torch.equal(t.bbox[pos].cpu(), torch.from_numpy(bbs.astype(np.int16)))
        got_sample.append(ids64[ids64 % 100 == 0])
        del t
    got = np.concatenate(got_sample)
    want = sample_ids[V.all(axis=0)]
    assert np.array_equal(got, want)
