"""Oracle cache writer for the full-size parity tests (TEST INFRASTRUCTURE: calls only oracle/
and the input generator synth/; never the CUDA path).

For one workload it writes ``tests/golden/cache/<key>.npz`` (``key`` = ``Workload.key``):

* the bbox redraw table (R12 "near-threshold tuples excluded by
  construction"): every covered tuple whose oracle margin ``z_target - max_{c != target} z_c``
  is below ``DELTA`` = 0.05 in absolute value for ANY classifier head of the workload gets its
  bbox redrawn (retry counter + 1, ``synth.make_tuples``) until every margin is >= DELTA;
* the oracle verdict matrix ``V[k, i] = p_k(t_i)`` of the covered tuples (every predicate on
  every tuple, no short-circuit), from which the tests derive the expected rows
  (``oracle.query_result``) and every per-batch counter (``oracle.sequential_eval``);
* the smallest |margin| per classifier head (>= DELTA by construction).

Covered tuples: ids [0, n) ("prefix") or the deterministic 1 % sample id % 100 == 0 of [0, n)
("mod100", cfg5; SURVEY.md §8(d) "Coverage").

    python -m tests.oracle_cache cfg2 [--weights bf16] [--small] [--n N] [--mode mod100] [--procs 8]
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from synth import workload  # noqa: E402
from synth.workload import CACHE_DIR, GEN_VERSION  # noqa: E402

DELTA = 0.05     # guaranteed |margin| of every classifier head
CHUNK = 4096     # tuples per worker task
SUB = 512        # tuples per crop matrix

_G = {}


def _init(threads: int):
    from threadpoolctl import threadpool_limits
    threadpool_limits(threads)


def _classifiers(w):
    return [k for k, p in enumerate(w.preds) if p["kind"] in ("linear", "mlp")]


def _eval(args):
    """Verdicts of every predicate and the margins of the classifier heads for the tuples `ids`
    drawn with redraw counters `retry`."""
    ids, retry = args
    w, fr = _G["w"], _G["frames"]
    w.redraw = (ids, retry)
    tup = O.as_numpy_tuples(w.tuples_at(ids))
    P, n = len(w.preds), len(ids)
    V = np.zeros((P, n), dtype=bool)
    M = np.full((P, n), np.inf)
    for a in range(0, n, SUB):
        sl = slice(a, min(a + SUB, n))
        fid, bb = tup["frame_id"][sl], tup["bbox"][sl]
        crops = {}
        for k, p in enumerate(w.preds):
            if p["kind"] in ("linear", "mlp"):
                mode = p.get("crop_mode", "nearest")
                if mode not in crops:
                    crops[mode] = O.crop_features(p, fr, fid, bb)
                z = (O.mlp_logits if p["kind"] == "mlp" else O.linear_logits)(p, crops[mode])
                V[k, sl] = O.argmax_first(z) == int(p["target"])
                M[k, sl] = O.margin(z, int(p["target"]))
            elif p["kind"] == "hsv":
                V[k, sl] = O.hsv_verdict(p, fr, fid, bb)
            else:
                sub = {key: col[sl] for key, col in tup.items()}
                V[k, sl] = O.predicate_verdict(p, sub)
    return V, M


def compute(w, ids: np.ndarray, procs: int = 8, verbose: bool = False, frames: np.ndarray = None):
    """(retry, V, min |margin| per predicate) for the tuples `ids` of workload `w`: the redraw loop of
    the module docstring, then the verdicts of every predicate on the final tuples."""
    _G["w"] = w
    _G["frames"] = frames if frames is not None else (w.frames().numpy() if w.needs_frames else None)
    retry = np.zeros(len(ids), dtype=np.int64)
    P = len(w.preds)
    V = np.zeros((P, len(ids)), dtype=bool)
    min_m = np.full(P, np.inf)
    cls = _classifiers(w)
    todo = np.arange(len(ids))
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_init, initargs=(1,)) as pool:
        it = 0
        while len(todo):
            tasks = [(ids[todo[a:a + CHUNK]], retry[todo[a:a + CHUNK]]) for a in range(0, len(todo), CHUNK)]
            res = pool.map(_eval, tasks, chunksize=1)
            Vt = np.concatenate([r[0] for r in res], axis=1)
            Mt = np.concatenate([r[1] for r in res], axis=1)
            V[:, todo] = Vt
            bad = np.zeros(len(todo), dtype=bool)
            for k in cls:
                bad |= np.abs(Mt[k]) < DELTA
            if verbose:
                print(f"[{w.name}] pass {it}: {len(todo)} tuples, {int(bad.sum())} redrawn "
                      f"({time.time() - t0:.0f} s)", flush=True)
            retry[todo[bad]] += 1
            todo = todo[bad]
            it += 1
            if it > 64:
                raise RuntimeError("redraw did not converge")
        if cls:  # the final margins of every covered tuple (the last evaluation of each one)
            res = pool.map(_eval, [(ids[a:a + CHUNK], retry[a:a + CHUNK]) for a in range(0, len(ids), CHUNK)],
                           chunksize=1)
            Vf = np.concatenate([r[0] for r in res], axis=1)
            Mf = np.concatenate([r[1] for r in res], axis=1)
            assert np.array_equal(Vf, V)
            for k in cls:
                min_m[k] = float(np.abs(Mf[k]).min()) if len(ids) else np.inf
                assert min_m[k] >= DELTA
    return retry, V, min_m


def make_safe(w, n: int, procs: int = 4):
    """In memory (tests): redraws the bboxes of w's first n tuples until every classifier margin is
    >= DELTA and installs the table as w.redraw; returns the oracle verdicts V of those tuples."""
    ids = np.arange(n, dtype=np.int64)
    w.redraw = None
    retry, V, _ = compute(w, ids, procs)
    nz = retry > 0
    w.redraw = (ids[nz], retry[nz])
    return V


def build(name: str, weights: str = "grid", small: bool = False, n: int = None, mode: str = "prefix",
          procs: int = 8, out_dir: str = CACHE_DIR, verbose: bool = True) -> str:
    w = workload(name, n=n, small=small, weights=weights, redraw=False)
    N = w.n
    ids = np.arange(0, N, 100 if mode == "mod100" else 1, dtype=np.int64)
    t0 = time.time()
    retry, V, min_m = compute(w, ids, procs, verbose)
    nz = retry > 0
    meta = dict(name=name, weights=weights, small=small, n=N, mode=mode, covered=int(len(ids)),
                gen_version=GEN_VERSION, delta=DELTA, preds=[p.get("name", p["kind"]) for p in w.preds],
                min_abs_margin=[None if not np.isfinite(m) else m for m in min_m.tolist()],
                redrawn=int(nz.sum()), max_retry=int(retry.max(initial=0)),
                selectivity=[float(v) for v in V.mean(axis=1)], results=int(V.all(axis=0).sum()),
                written_by="python -m tests.oracle_cache " + " ".join(sys.argv[1:]), seconds=round(time.time() - t0))
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, w.key + ".npz")
    np.savez_compressed(path, meta=np.array(json.dumps(meta)), redraw_ids=ids[nz], redraw_retry=retry[nz].astype(np.uint8),
                        V_bits=np.packbits(V, axis=1), covered_ids=ids if mode != "prefix" else np.zeros(0, np.int64))
    if verbose:
        print(json.dumps(meta))
    return path


def load(key: str):
    """(meta, covered ids, V) of a cache file."""
    with np.load(os.path.join(CACHE_DIR, key + ".npz")) as z:
        meta = json.loads(str(z["meta"]))
        n = meta["covered"]
        V = np.unpackbits(z["V_bits"], axis=1, count=n).astype(bool)
        ids = z["covered_ids"] if meta["mode"] != "prefix" else np.arange(n, dtype=np.int64)
    return meta, ids, V


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--weights", default="grid", choices=["grid", "bf16"])
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--mode", default="prefix", choices=["prefix", "mod100"])
    ap.add_argument("--procs", type=int, default=8)
    a = ap.parse_args()
    print(build(a.name, a.weights, a.small, a.n, a.mode, a.procs))
