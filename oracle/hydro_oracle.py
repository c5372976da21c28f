"""Plain, slow, obviously-correct CPU oracle for Hydro's eddy hot path (arXiv 2403.14902).

TEST INFRASTRUCTURE ONLY -- imported solely by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  It shares no code with the CUDA
path (paper_2403_14902_b200/) and imports nothing from it.  Inputs come from
``synth`` (which holds no method arithmetic).  Arithmetic is float64 numpy unless
the method fixes another precision (bf16 crop values, f32 area division).

What it computes (PAPER.md citations; "R<n>" = numbered reading in DESIGN.md §2):

* the query result: ``SELECT id, bbox ... WHERE p_1 AND ... AND p_P`` (PAPER.md:43-49,
  276-282) -- every predicate evaluated on every tuple, no short-circuit, rows kept in
  input (ascending id) order (R18);
* per-predicate verdicts, each a pure function of the tuple:
  LABEL_EQ, HASH (R5, stand-in for the synthetic 10/20 ms predicates,
  PAPER.md:550-552), LINEAR = argmax(W . Crop(frame, bbox) + b) == target (PAPER.md:47-48,
  286-288; R9-R14, R19), MLP = argmax(W2 . bf16(relu(W1 . Crop + b1)) + b2) == target (R25);
* eddy statistics: count-based selectivity, measured cost,
  the score ``cost / (1 - selectivity)`` and its lowest-first order,
  the decayed fold (R4), the closed-form expected cost (R20);
* the sequential short-circuit evaluation with eager materialization (PAPER.md:227,
  251-253) used to pin order independence and the STATIC counters.

Pins: tests/test_oracle.py checks every function here against something other than
itself (published hash vectors, torch's interpolate / adaptive_avg_pool2d, one-hot and
constant-frame closed forms, brute force over all orders, the paper's printed numbers).
Parity unpinned: none of the functions below.  Measured cycle costs (an input to the
fold) are not reproducible and are taken from the GPU's own report (DESIGN.md §2 R6).
"""
from __future__ import annotations

import itertools
import math
from typing import Dict, List, Sequence

import numpy as np

CROP = 64
K_FEATURES = CROP * CROP * 3

# --------------------------------------------------------------------------------------
# HASH predicate (R5): SplitMix64 (Steele/Lea/Flood) + murmur3 fmix32 rounds.

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_SM_M1 = np.uint64(0xBF58476D1CE4E5B9)
_SM_M2 = np.uint64(0x94D049BB133111EB)
_FM_M1 = np.uint32(0x85EBCA6B)
_FM_M2 = np.uint32(0xC2B2AE35)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """z = x + golden; z = (z ^ z>>30) * M1; z = (z ^ z>>27) * M2; return z ^ z>>31 (mod 2**64)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _SM_M1
        z = (z ^ (z >> np.uint64(27))) * _SM_M2
        return z ^ (z >> np.uint64(31))


def fmix32(h: np.ndarray) -> np.ndarray:
    """murmur3 finaliser: h^=h>>16; h*=0x85EBCA6B; h^=h>>13; h*=0xC2B2AE35; h^=h>>16 (mod 2**32)."""
    h = np.asarray(h, dtype=np.uint32)
    with np.errstate(over="ignore"):
        h = h ^ (h >> np.uint32(16))
        h = h * _FM_M1
        h = h ^ (h >> np.uint32(13))
        h = h * _FM_M2
        return h ^ (h >> np.uint32(16))


def bbox_wh(bbox: np.ndarray):
    b = np.asarray(bbox, dtype=np.int64)
    return b[:, 2] - b[:, 0], b[:, 3] - b[:, 1]


def hash_units(pred: Dict, bbox: np.ndarray) -> np.ndarray:
    """units(t) = units, or ceil(w*h / units_per_area) when units_per_area > 0 (cfg4)."""
    n = len(bbox)
    if pred.get("units_per_area", 0) > 0:
        w, h = bbox_wh(bbox)
        upa = int(pred["units_per_area"])
        return np.maximum((w * h + upa - 1) // upa, 1)
    return np.full(n, int(pred["units"]), dtype=np.int64)


def hash_verdict(pred: Dict, ids: np.ndarray, bbox: np.ndarray) -> np.ndarray:
    """v(t): h = hi32(splitmix64(id ^ seed)); for r < units(t): h = fmix32(h + r); h < T(t)."""
    ids = np.asarray(ids, dtype=np.uint64)
    units = hash_units(pred, bbox)
    h = (splitmix64(ids ^ np.uint64(pred["seed"])) >> np.uint64(32)).astype(np.uint32)
    with np.errstate(over="ignore"):
        for r in range(int(units.max(initial=0))):
            h = np.where(r < units, fmix32(h + np.uint32(r)), h)
    t0, t1 = pred["threshold"]
    T = np.where(ids >= np.uint64(pred["drift_id"]), np.uint64(t1), np.uint64(t0))
    return h.astype(np.uint64) < T


def label_verdict(pred: Dict, label: np.ndarray) -> np.ndarray:
    """Object.label = 'dog'."""
    return np.asarray(label).astype(np.int64) == int(pred["label"])


# --------------------------------------------------------------------------------------
# Crop(frame, bbox) -> 64x64x3 (size and interpolation: R10)


def crop_nearest(frames: np.ndarray, frame_id: np.ndarray, bbox: np.ndarray) -> np.ndarray:
    """NEAREST_EXACT: sy = y0 + ((2dy+1)h) // 128, sx = x0 + ((2dx+1)w) // 128; -> uint8 [n,64,64,3]."""
    b = np.asarray(bbox, dtype=np.int64)
    x0, y0 = b[:, 0], b[:, 1]
    w, h = bbox_wh(b)
    d = np.arange(CROP, dtype=np.int64)
    sy = y0[:, None] + ((2 * d[None, :] + 1) * h[:, None]) // (2 * CROP)
    sx = x0[:, None] + ((2 * d[None, :] + 1) * w[:, None]) // (2 * CROP)
    f = np.asarray(frame_id, dtype=np.int64)
    return frames[f[:, None, None], sy[:, :, None], sx[:, None, :]]


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (nearest, ties to even); returned as float32 holding the bf16 value."""
    bits = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    bias = np.uint64(0x7FFF) + ((bits >> np.uint64(16)) & np.uint64(1))
    r = ((bits + bias) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32)


def crop_area(frames: np.ndarray, frame_id: np.ndarray, bbox: np.ndarray) -> np.ndarray:
    """AREA: bin [y0 + dy*h//64, y0 + ceil((dy+1)h/64)) x same in x; value = bf16_rne(f32(sum)/f32(count)).

    Returns float32 [n,64,64,3] holding bf16 values (R10, R19).  Sums are exact int64.
    """
    b = np.asarray(bbox, dtype=np.int64)
    out = np.empty((len(b), CROP, CROP, 3), dtype=np.float32)
    d = np.arange(CROP, dtype=np.int64)
    for i in range(len(b)):
        x0, y0, x1, y1 = (int(v) for v in b[i])
        w, h = x1 - x0, y1 - y0
        img = frames[int(frame_id[i]), y0:y1, x0:x1, :].astype(np.int64)
        sat = np.zeros((h + 1, w + 1, 3), dtype=np.int64)  # summed-area table
        sat[1:, 1:] = img.cumsum(0).cumsum(1)
        ys, ye = (d * h) // CROP, ((d + 1) * h + CROP - 1) // CROP
        xs, xe = (d * w) // CROP, ((d + 1) * w + CROP - 1) // CROP
        s = (sat[ye[:, None], xe[None, :]] - sat[ys[:, None], xe[None, :]]
             - sat[ye[:, None], xs[None, :]] + sat[ys[:, None], xs[None, :]])
        cnt = ((ye - ys)[:, None] * (xe - xs)[None, :])[:, :, None]
        out[i] = f32_to_bf16_rne(s.astype(np.float32) / cnt.astype(np.float32))
    return out


def crop_features(pred: Dict, frames, frame_id, bbox) -> np.ndarray:
    """x[(dy*64+dx)*3+ch] (HWC flatten of the crop; R10) as float64 [n, 12288]."""
    if pred.get("crop_mode", "nearest") == "area":
        c = crop_area(frames, frame_id, bbox)
    else:
        c = crop_nearest(frames, frame_id, bbox)
    return c.reshape(len(bbox), K_FEATURES).astype(np.float64)


# --------------------------------------------------------------------------------------
# LINEAR classifier predicate (stand-in for DogBreed/DogColorClassifier, R12-R14)


def linear_logits(pred: Dict, x: np.ndarray) -> np.ndarray:
    """z_c = sum_k x_k W[c][k] + b[c] in float64 from the exact bf16 W and f32 b."""
    W = np.asarray(pred["weight"].float().numpy() if hasattr(pred["weight"], "float") else pred["weight"],
                   dtype=np.float64)
    b = np.asarray(pred["bias"].numpy() if hasattr(pred["bias"], "numpy") else pred["bias"],
                   dtype=np.float64)
    return x @ W.T + b[None, :]


def _f64(t) -> np.ndarray:
    if hasattr(t, "float"):
        return t.float().cpu().numpy().astype(np.float64)
    return np.asarray(t, dtype=np.float64)


def mlp_logits(pred: Dict, x: np.ndarray) -> np.ndarray:
    """MLP head (R25, the north star's "small ... MLP classifier"):

    a = W1 x + b1                       (float64; the method accumulates in fp32)
    h = bf16_rne(f32(max(a, 0)))        (the hidden layer is bf16, as the second GEMM's operand)
    z = W2 h + b2                       (float64 from the exact bf16 h, W2 and f32 b2)
    """
    W1, b1 = _f64(pred["weight"]), _f64(pred["bias"])
    W2, b2 = _f64(pred["weight2"]), _f64(pred["bias2"])
    a = x @ W1.T + b1[None, :]
    h = f32_to_bf16_rne(np.maximum(a, 0.0).astype(np.float32)).astype(np.float64)
    return h @ W2.T + b2[None, :]


# --------------------------------------------------------------------------------------
# HSV colour heuristic (DogColorClassifier; R27)

# inclusive (H, S, V) boxes in OpenCV's 8-bit convention (H in [0, 180), S, V in [0, 255]);
# class c is the union of its boxes; only red's range is printed in the paper
HSV_COLOURS = ["red", "black", "gray", "yellow", "green", "blue", "purple", "pink", "white", "other"]
HSV_BOXES = [
    [((0, 50, 70), (9, 255, 255)), ((170, 50, 70), (179, 255, 255))],  # red (PAPER.md:395 + hue wrap)
    [((0, 0, 0), (179, 255, 30))],                                     # black
    [((0, 0, 31), (179, 18, 230))],                                    # gray
    [((20, 50, 70), (34, 255, 255))],                                  # yellow
    [((35, 50, 70), (89, 255, 255))],                                  # green
    [((90, 50, 70), (128, 255, 255))],                                 # blue
    [((129, 50, 70), (158, 255, 255))],                                # purple
    [((159, 50, 70), (169, 255, 255))],                                # pink
    [((0, 0, 231), (179, 18, 255))],                                   # white
]


HSV_SHIFT = 12  # OpenCV's fixed-point shift for 8-bit RGB -> HSV


def _hsv_tables():
    """OpenCV's 8-bit reciprocal tables (R27): sdiv[i] = round(255 * 2^12 / i),
    hdiv[i] = round(180 * 2^12 / (6 i)) for i = 1..255, both 0 at i = 0 (no exact .5 occurs:
    2 * 255 * 2^12 / i and 2 * 180 * 2^12 / (6 i) are never odd integers for i < 2^13)."""
    i = np.arange(256, dtype=np.float64)
    sdiv = np.zeros(256, np.int64)
    hdiv = np.zeros(256, np.int64)
    sdiv[1:] = np.rint((255 << HSV_SHIFT) / i[1:])
    hdiv[1:] = np.rint((180 << HSV_SHIFT) / (6.0 * i[1:]))
    return sdiv, hdiv


def rgb_to_hsv_u8(rgb: np.ndarray) -> np.ndarray:
    """8-bit RGB -> 8-bit HSV exactly as OpenCV's cvtColor(COLOR_RGB2HSV) (R27; the paper's red
    range, is in OpenCV's H in [0, 180) scale), plain fixed-point steps:
      V = max(R, G, B), d = V - min(R, G, B)
      S = (d * sdiv[V] + 2^11) >> 12
      h = G - B if V == R, else B - R + 2d if V == G, else R - G + 4d
      H = (h * hdiv[d] + 2^11) >> 12 (floor shift), + 180 if negative.
    Pinned bit for bit against cv2.cvtColor on all 2^24 colours (tests/test_oracle.py)."""
    sdiv, hdiv = _hsv_tables()
    c = np.asarray(rgb, dtype=np.int64)
    R, G, B = c[..., 0], c[..., 1], c[..., 2]
    V = np.maximum(np.maximum(R, G), B)
    d = V - np.minimum(np.minimum(R, G), B)
    half = 1 << (HSV_SHIFT - 1)
    S = (d * sdiv[V] + half) >> HSV_SHIFT
    h = np.where(V == R, G - B, np.where(V == G, B - R + 2 * d, R - G + 4 * d))
    H = (h * hdiv[d] + half) >> HSV_SHIFT
    H = np.where(H < 0, H + 180, H)
    return np.stack([H, S, V], axis=-1)


def hsv_class(hsv: np.ndarray) -> np.ndarray:
    """Colour class per pixel: the first box containing it, else 9 ('other')."""
    out = np.full(hsv.shape[:-1], 9, dtype=np.int64)
    for c in range(len(HSV_BOXES) - 1, -1, -1):  # reverse so the lowest class index wins overlaps
        inside = np.zeros(hsv.shape[:-1], dtype=bool)
        for lo, hi in HSV_BOXES[c]:
            inside |= np.all((hsv >= np.array(lo)) & (hsv <= np.array(hi)), axis=-1)
        out = np.where(inside, c, out)
    return out


def hsv_counts(crops_u8: np.ndarray) -> np.ndarray:
    """Per crop the number of pixels of each of the 10 classes (crops [n, 64, 64, 3] u8)."""
    cls = hsv_class(rgb_to_hsv_u8(crops_u8)).reshape(len(crops_u8), -1)
    return np.stack([(cls == c).sum(axis=1) for c in range(10)], axis=1)


def hsv_verdict(pred: Dict, frames, frame_id, bbox, return_counts=False):
    """DogColorClassifier(Crop(frame, bbox)) = colour: the class with most pixels of the 64x64
    nearest crop (lowest index on ties) equals the target (R27)."""
    counts = hsv_counts(crop_nearest(frames, frame_id, bbox))
    v = argmax_first(counts.astype(np.float64)) == int(pred["target"])
    return (v, counts) if return_counts else v


def argmax_first(z: np.ndarray) -> np.ndarray:
    """argmax over classes, lowest index on ties (R12)."""
    best = np.zeros(z.shape[0], dtype=np.int64)
    for c in range(1, z.shape[1]):
        best = np.where(z[:, c] > z[np.arange(z.shape[0]), best], c, best)
    return best


def margin(z: np.ndarray, target: int) -> np.ndarray:
    """m = z_target - max_{c != target} z_c."""
    others = np.delete(z, target, axis=1)
    return z[:, target] - others.max(axis=1)


def linear_verdict(pred: Dict, frames, frame_id, bbox, chunk=512, return_logits=False):
    """LINEAR and MLP classifier predicates: argmax(logits(Crop(frame, bbox))) == target."""
    head = mlp_logits if pred["kind"] == "mlp" else linear_logits
    out, logits = [], []
    for a in range(0, len(bbox), chunk):
        x = crop_features(pred, frames, frame_id[a:a + chunk], bbox[a:a + chunk])
        z = head(pred, x)
        out.append(argmax_first(z) == int(pred["target"]))
        if return_logits:
            logits.append(z)
    v = np.concatenate(out) if out else np.zeros(0, dtype=bool)
    if return_logits:
        return v, (np.concatenate(logits) if logits else np.zeros((0, int(pred["n_classes"]))))
    return v


# --------------------------------------------------------------------------------------
# Evaluate-all and the query result ("iff it passes all filters")


def as_numpy_tuples(t) -> Dict[str, np.ndarray]:
    """Accepts synth.Tuples or a dict; returns numpy columns (id u64, frame_id, bbox int64, label)."""
    if isinstance(t, dict):
        return t
    return dict(id=t.id.cpu().numpy().astype(np.uint64), frame_id=t.frame_id.cpu().numpy().astype(np.int64),
                bbox=t.bbox.cpu().numpy().astype(np.int64), label=t.label.cpu().numpy().astype(np.int64))


def predicate_verdict(pred: Dict, tup: Dict[str, np.ndarray], frames=None) -> np.ndarray:
    kind = pred["kind"]
    if kind == "label_eq":
        return label_verdict(pred, tup["label"])
    if kind == "hash":
        return hash_verdict(pred, tup["id"], tup["bbox"])
    if kind in ("linear", "mlp"):
        return linear_verdict(pred, frames, tup["frame_id"], tup["bbox"])
    if kind == "hsv":
        return hsv_verdict(pred, frames, tup["frame_id"], tup["bbox"])
    raise ValueError(kind)


def evaluate_all(preds: Sequence[Dict], tuples, frames=None) -> np.ndarray:
    """Verdict matrix V[k, i] = p_k(t_i) for every predicate and every tuple (no short-circuit)."""
    tup = as_numpy_tuples(tuples)
    n = len(tup["id"])
    V = np.zeros((len(preds), n), dtype=bool)
    for k, p in enumerate(preds):
        V[k] = predicate_verdict(p, tup, frames)
    return V


def query_result(tuples, V: np.ndarray):
    """R = [(id, bbox) for t in tuples if AND_k V[k, t]] in input order."""
    tup = as_numpy_tuples(tuples)
    keep = np.all(V, axis=0) if len(V) else np.ones(len(tup["id"]), dtype=bool)
    return tup["id"][keep], tup["bbox"][keep], keep


# --------------------------------------------------------------------------------------
# Eager-materialization short-circuit evaluation of one routing batch in a given order
# ("dropped immediately", 251-253)


def sequential_eval(V: np.ndarray, order: Sequence[int]):
    """Run predicates in ``order`` on the alive set only; returns (in_k, pass_k, alive mask)."""
    P, n = V.shape
    alive = np.ones(n, dtype=bool)
    n_in = np.zeros(P, dtype=np.int64)
    n_pass = np.zeros(P, dtype=np.int64)
    for k in order:
        n_in[k] = int(alive.sum())
        alive = alive & V[k]
        n_pass[k] = int(alive.sum())
    return n_in, n_pass, alive


# --------------------------------------------------------------------------------------
# Statistics, score, order (R1-R4, R20)


def selectivity(s_in: float, s_pass: float, prior: float = 0.5) -> float:
    """passed / in; prior when nothing observed (R3)."""
    return prior if s_in <= 0 else s_pass / s_in


def cost_per_tuple(s_in: float, s_cost: float, declared: float) -> float:
    """cost / in (PAPER.md:248, 422 'ms per tuple'); declared cost when nothing observed (R3)."""
    return declared if s_in <= 0 else s_cost / s_in


def score(c: float, s: float) -> float:
    """Hellerstein rank c / (1 - s): 0 when c == 0, +inf when s >= 1 (R1)."""
    if c == 0.0:
        return 0.0
    if s >= 1.0:
        return math.inf
    return c / (1.0 - s)


def policy_key(policy: str, c: float, s: float) -> float:
    """score-driven (default), cost-driven, selectivity-driven."""
    if policy in ("score", "static"):
        return score(c, s)
    if policy == "cost":
        return c
    if policy == "selectivity":
        return s
    raise ValueError(policy)


def reuse_estimated_cost(c: float, hit: float) -> float:
    """Reuse-aware routing: estimated cost = (1 - cache hit rate) * cost of
    computing the UDF; the cache lookup is assumed free."""
    return (1.0 - hit) * c


def cache_hit_rate(ids: np.ndarray, cached: Sequence[tuple]) -> float:
    """Fraction of a batch's tuple ids whose verdict is cached; ``cached`` = open id intervals
    (lo, hi) as in UC2's ``WHERE id > lo AND id < hi``."""
    ids = np.asarray(ids, dtype=np.int64)
    if len(ids) == 0:
        return 0.0
    hit = np.zeros(len(ids), dtype=bool)
    for lo, hi in cached:
        hit |= (ids > lo) & (ids < hi)
    return float(hit.mean())


def reuse_order(costs: Sequence[float], hits: Sequence[float]) -> List[int]:
    """Lowest estimated cost first, ties -> lowest predicate id (R2)."""
    return order_by_key([reuse_estimated_cost(c, h) for c, h in zip(costs, hits)])


def order_by_key(keys: Sequence[float]) -> List[int]:
    """Lowest key first; ties -> lowest predicate id (R2)."""
    return sorted(range(len(keys)), key=lambda k: (keys[k], k))


def expected_cost(order: Sequence[int], c: Sequence[float], s: Sequence[float]) -> float:
    """E(pi) = sum_i c_{pi_i} * prod_{j<i} s_{pi_j} per input tuple (independent predicates, R20)."""
    e, p = 0.0, 1.0
    for k in order:
        e += c[k] * p
        p *= s[k]
    return e


def realized_cost(n_in: Sequence[int], c: Sequence[float]) -> float:
    """sum_k c_k * in_k."""
    return float(sum(ci * ni for ci, ni in zip(c, n_in)))


class FoldState:
    """Decayed statistics S <- gamma*S + delta, applied per predicate only when delta_in > 0 (R4).

    gamma = 1 gives the paper's plain cumulative counts.
    """

    def __init__(self, n_pred: int, gamma: float, declared_cost: Sequence[float], prior: float = 0.5,
                 cost_source: str = "measured"):
        self.cost_source = cost_source  # "declared": c is always the declared cost (R6)
        self.s_in = [0.0] * n_pred
        self.s_pass = [0.0] * n_pred
        self.s_cost = [0.0] * n_pred
        self.gamma = gamma
        self.declared = list(declared_cost)
        self.prior = prior

    def fold(self, d_in, d_pass, d_cost):
        for k in range(len(self.s_in)):
            if d_in[k] > 0:
                self.s_in[k] = self.gamma * self.s_in[k] + float(d_in[k])
                self.s_pass[k] = self.gamma * self.s_pass[k] + float(d_pass[k])
                self.s_cost[k] = self.gamma * self.s_cost[k] + float(d_cost[k])

    def sel(self):
        return [selectivity(a, b, self.prior) for a, b in zip(self.s_in, self.s_pass)]

    def cost(self):
        if self.cost_source == "declared":
            return list(self.declared)
        return [cost_per_tuple(a, c, d) for a, c, d in zip(self.s_in, self.s_cost, self.declared)]

    def order(self, policy="score"):
        c, s = self.cost(), self.sel()
        return order_by_key([policy_key(policy, ci, si) for ci, si in zip(c, s)])


def brute_force_best_orders(c: Sequence[float], s: Sequence[float]):
    """All orders minimising E(pi) (exhaustive, for pins on tiny inputs)."""
    best, arg = math.inf, []
    for perm in itertools.permutations(range(len(c))):
        e = expected_cost(perm, c, s)
        if e < best - 1e-12 * max(1.0, abs(best) if best < math.inf else 1.0):
            best, arg = e, [perm]
        elif abs(e - best) <= 1e-12 * max(1.0, abs(best)):
            arg.append(perm)
    return best, arg


# ------------------------------------------------------------------------------------------
# Data-aware load balancing (R28).
# The Laminar router gives work to the least-loaded worker, the load being estimated
# proactively from the input size ("input size as a reasonable proxy for execution cost ...
# for vision models, it is the input image/frame size").  For a classifier
# hop the workers are the G persistent CTAs; the hop's input (positions 0..count-1) is cut into
# G contiguous ranges of equal estimated cost, at 32-position granularity (R28).

def input_size_costs(bbox: np.ndarray) -> np.ndarray:
    """Estimated cost of each tuple = its input size w * h."""
    w, h = bbox_wh(bbox)
    return (w * h).astype(np.int64)


def chunk_costs(costs: np.ndarray, chunk: int = 32) -> np.ndarray:
    """Sum of the estimated costs over consecutive `chunk`-position chunks (last one ragged)."""
    n = len(costs)
    out = np.zeros((n + chunk - 1) // chunk, np.int64)
    for k in range(len(out)):
        out[k] = int(costs[k * chunk:(k + 1) * chunk].sum())
    return out


def balanced_bounds(chunk_cost: np.ndarray, G: int, count: int, chunk: int = 32) -> List[int]:
    """R28: worker c (0 <= c < G) starts at chunk min{k : X_k * G >= c * A}, X_k the cost of the
    chunks before k and A the total; bounds[0] = 0, bounds[G] = count, positions clipped to
    count.  Each worker's load is at most A / G plus one chunk.  Plain loops, exact integers."""
    A = int(sum(int(x) for x in chunk_cost))
    bounds = [0] * (G + 1)
    bounds[G] = count
    if A == 0:
        return bounds
    X = [0]
    for x in chunk_cost:
        X.append(X[-1] + int(x))  # X[k] = exclusive prefix of chunk k; X[n] = A
    for c in range(1, G):
        k = next(k for k in range(len(X)) if X[k] * G >= c * A)
        bounds[c] = min(chunk * k, count)
    return bounds


def range_loads(costs: np.ndarray, bounds: Sequence[int]) -> List[int]:
    """Estimated load of every worker for position ranges [bounds[c], bounds[c+1])."""
    return [int(costs[bounds[c]:bounds[c + 1]].sum()) for c in range(len(bounds) - 1)]


def round_robin_loads(costs: np.ndarray, G: int, tile: int = 128) -> List[int]:
    """Estimated load of every worker when tile i (128 positions) goes to worker i mod G, the
    default round-robin routing."""
    loads = [0] * G
    for i in range((len(costs) + tile - 1) // tile):
        loads[i % G] += int(costs[i * tile:(i + 1) * tile].sum())
    return loads


# ------------------------------------------------------------------------------------------
# Concurrent workers and cost-driven routing (
# DESIGN.md R29).  Each predicate runs on its own resource ("worker"), serially FIFO; an item
# enters predicate i+1 when predicate i passed it (eager materialization).

def two_stage_completion(n_items: int, cost_first: float, cost_second: float, pass_mask) -> float:
    """The timeline of Fig. cost_route: item i (1-indexed) leaves stage 1 at
    i * cost_first; a passing item queues for stage 2, which serves one item at a time for
    cost_second each.  Returns the completion instant of the last event of either stage."""
    t1 = 0.0
    t2 = 0.0
    for i in range(n_items):
        t1 += cost_first
        if pass_mask[i]:
            t2 = max(t2, t1) + cost_second
    return max(t1, t2)


def flow_shop_makespan(stage_times) -> float:
    """Batches through P serial workers in a fixed order (a permutation flow shop): batch b's
    stage i starts when its stage i-1 and batch b-1's stage i are done,
    C[b][i] = max(C[b][i-1], C[b-1][i]) + t[b][i]; returns C[last][last].  With one item per
    batch and P = 2 it is two_stage_completion."""
    prev = None
    for row in stage_times:
        cur = []
        for i, t in enumerate(row):
            start = max(cur[i - 1] if i else 0.0, prev[i] if prev is not None else 0.0)
            cur.append(start + float(t))
        prev = cur
    return prev[-1] if prev else 0.0


def pipeline_stage_times(V: np.ndarray, order: Sequence[int], batch: int, time_per_tuple: Sequence[float]):
    """Stage times of every routing batch when the batch visits the workers in `order`: stage i
    sees the tuples that passed the earlier stages (oracle verdicts V[k, t]) and costs
    time_per_tuple[order[i]] per tuple."""
    out = []
    n = V.shape[1]
    for a in range(0, n, batch):
        Vb = V[:, a:a + batch]
        alive = np.ones(Vb.shape[1], dtype=bool)
        row = []
        for k in order:
            row.append(int(alive.sum()) * float(time_per_tuple[k]))
            alive &= Vb[k]
        out.append(row)
    return out
