"""Pins for the CPU oracle (-m "not gpu").  Each test checks oracle/ against something other
than itself: published hash vectors, torch's interpolate / adaptive_avg_pool2d, closed forms,
brute force over all orders, and numbers printed in PAPER.md (tests/golden/paper_pins.json).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
from synth import Tuples, hash_pred, make_frames, make_tuples, workload
from synth.workload import WEIGHT_SCALE

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


# ----------------------------------------------------------------------------- HASH (R5)

def test_splitmix64_published_sequence():
    g = 0x9E3779B97F4A7C15
    seq = [int(O.splitmix64(np.uint64((i * g) % 2 ** 64))) for i in range(3)]
    assert seq == [int(v, 16) for v in GOLD["hash_vectors"]["splitmix64_seq0"]]


def test_fmix32_published_vectors():
    for k, v in GOLD["hash_vectors"]["fmix32"].items():
        assert int(O.fmix32(np.uint32(int(k, 16)))) == int(v, 16)


@pytest.mark.parametrize("sel", [0.1, 0.5, 0.9, 0.254])
@pytest.mark.parametrize("units", [1, 4])
def test_hash_selectivity_binomial_band(sel, units):
    n = 200_000
    p = hash_pred(7, sel, units=units)
    ids = np.arange(n, dtype=np.uint64)
    bbox = np.tile(np.array([[0, 0, 8, 8]]), (n, 1))
    rate = O.hash_verdict(p, ids, bbox).mean()
    assert abs(rate - sel) < 5 * math.sqrt(sel * (1 - sel) / n)


def test_hash_threshold_extremes_and_drift():
    ids = np.arange(1000, dtype=np.uint64)
    bbox = np.tile(np.array([[0, 0, 8, 8]]), (1000, 1))
    assert O.hash_verdict(hash_pred(3, 1.0), ids, bbox).all()      # T = 2**32 passes all
    assert not O.hash_verdict(hash_pred(3, 0.0), ids, bbox).any()  # T = 0 passes none
    p = hash_pred(3, 1.0, sel_after=0.0, drift_id=500)
    v = O.hash_verdict(p, ids, bbox)
    assert v[:500].all() and not v[500:].any()


def test_hash_rounds_are_fmix_of_plus_r():
    # units = 2 is fmix32(fmix32(h0 + 0) + 1) with h0 = hi32(splitmix64(id ^ seed)), written out
    # independently with Python ints.
    seed, i = 99, 12345
    M64, M32 = 2 ** 64 - 1, 2 ** 32 - 1

    def sm(x):
        z = (x + 0x9E3779B97F4A7C15) & M64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def fm(h):
        h ^= h >> 16; h = (h * 0x85EBCA6B) & M32; h ^= h >> 13; h = (h * 0xC2B2AE35) & M32
        return h ^ (h >> 16)

    h = fm((fm(sm(i ^ seed) >> 32) + 1) & M32)
    for T in (h, h + 1):
        p = dict(kind="hash", seed=seed, threshold=(T, T), drift_id=2 ** 63 - 1, units=2, units_per_area=0)
        assert bool(O.hash_verdict(p, np.array([i], np.uint64), np.array([[0, 0, 1, 1]]))[0]) == (h < T)


def test_hash_units_per_area():
    p = hash_pred(5, 0.5, units_per_area=4096)
    bbox = np.array([[0, 0, 64, 64], [0, 0, 65, 64], [0, 0, 1, 1], [0, 0, 256, 256]])
    assert O.hash_units(p, bbox).tolist() == [1, 2, 1, 16]


def test_cfg1_counts():
    g = GOLD["cfg1_counts"]
    w = workload("cfg1")
    V = O.evaluate_all(w.preds, w.tuples())
    assert V[0].sum() == g["A_pass"] and V[1].sum() == g["B_pass"] and V.all(0).sum() == g["A_and_B"]
    n_in, n_pass, _ = O.sequential_eval(V, [0, 1])
    assert n_in.tolist() == [10000, g["A_pass"]] and n_pass.tolist() == [g["A_pass"], g["A_and_B"]]
    # realized cost of the run = 10000 * 1 + 5039 * 10 units (SURVEY.md §8(c) "realized 60,390")
    assert O.realized_cost(n_in, [1.0, 10.0]) == 60390.0


def test_realized_cost_equals_per_tuple_short_circuit_brute_force():
    """sum_k c_k in_k equals the cost summed tuple by tuple over a plain short-circuit AND (each
    tuple pays c_k for every predicate it reaches), for every order of random verdicts."""
    rng = np.random.default_rng(5)
    V = rng.random((4, 300)) < np.array([0.2, 0.5, 0.7, 0.9])[:, None]
    c = [3.0, 1.5, 7.0, 0.25]
    for order in itertools.permutations(range(4)):
        n_in, _, _ = O.sequential_eval(V, order)
        brute = 0.0
        for t in range(V.shape[1]):
            for k in order:
                brute += c[k]
                if not V[k, t]:
                    break
        assert O.realized_cost(n_in, c) == pytest.approx(brute, rel=1e-12)


# ----------------------------------------------------------------------------- crops (R10)

def _torch_crop(frame, b):
    x0, y0, x1, y1 = (int(v) for v in b)
    return torch.from_numpy(frame[y0:y1, x0:x1, :].copy()).permute(2, 0, 1)[None].double()


def test_crop_nearest_matches_torch_nearest_exact():
    F = make_frames(3, 4, 96, 128).numpy()
    t = make_tuples(3, 0, 300, n_frames=4, frame_h=96, frame_w=128, w_min=8, n_octaves=4)
    tup = O.as_numpy_tuples(t)
    mine = O.crop_nearest(F, tup["frame_id"], tup["bbox"])
    for i in range(len(tup["id"])):
        ref = torch.nn.functional.interpolate(_torch_crop(F[tup["frame_id"][i]], tup["bbox"][i]),
                                              size=(64, 64), mode="nearest-exact")
        assert np.array_equal(mine[i], ref[0].permute(1, 2, 0).numpy().astype(np.uint8))


def test_bf16_rounding_matches_torch():
    x = np.random.default_rng(0).standard_normal(100_000).astype(np.float32) * 300
    x = np.concatenate([x, np.float32([0.5, 1.5, 127.75, 255.0, 1 / 3, 2 / 3])])
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(O.f32_to_bf16_rne(x), ref)


def test_crop_area_matches_adaptive_avg_pool():
    F = make_frames(4, 3, 96, 128).numpy()
    t = make_tuples(4, 0, 60, n_frames=3, frame_h=96, frame_w=128, w_min=8, n_octaves=4)
    tup = O.as_numpy_tuples(t)
    mine = O.crop_area(F, tup["frame_id"], tup["bbox"])
    worst = 0.0
    for i in range(len(tup["id"])):
        ref = torch.nn.functional.adaptive_avg_pool2d(_torch_crop(F[tup["frame_id"][i]], tup["bbox"][i]), 64)
        ref = ref[0].permute(1, 2, 0).numpy()
        # exact mean vs the f32 division + bf16 rounding: within half a bf16 ulp (+ f32 slack)
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        worst = max(worst, float(np.max(np.abs(mine[i] - ref) / ulp)))
    assert worst <= 0.5 + 1e-3


# ----------------------------------------------------------------------------- LINEAR (R12)

def test_logits_one_hot_rows_select_crop_pixels():
    """W[c] = e_{k_c} -> z_c = x[k_c] + b_c; k = (dy*64+dx)*3+ch; x from torch nearest-exact."""
    F = make_frames(5, 2, 96, 128).numpy()
    t = make_tuples(5, 0, 40, n_frames=2, frame_h=96, frame_w=128, w_min=8, n_octaves=4)
    tup = O.as_numpy_tuples(t)
    picks = [(0, 0, 0), (0, 63, 2), (63, 0, 1), (17, 42, 2), (63, 63, 0), (31, 5, 1)]
    W = np.zeros((len(picks), O.K_FEATURES), np.float32)
    for c, (dy, dx, ch) in enumerate(picks):
        W[c, (dy * 64 + dx) * 3 + ch] = 1.0
    b = np.arange(len(picks), dtype=np.float32) * 0.5
    pred = dict(kind="linear", weight=torch.from_numpy(W).to(torch.bfloat16), bias=torch.from_numpy(b),
                target=0, n_classes=len(picks), crop_mode="nearest")
    z = O.linear_logits(pred, O.crop_features(pred, F, tup["frame_id"], tup["bbox"]))
    for i in range(len(tup["id"])):
        ref = torch.nn.functional.interpolate(_torch_crop(F[tup["frame_id"][i]], tup["bbox"][i]),
                                              size=(64, 64), mode="nearest-exact")[0]
        for c, (dy, dx, ch) in enumerate(picks):
            assert z[i, c] == float(ref[ch, dy, dx]) + b[c]


def test_logits_constant_frame_closed_form():
    F = np.full((1, 96, 128, 3), 7, np.uint8)
    t = make_tuples(6, 0, 10, n_frames=1, frame_h=96, frame_w=128, w_min=8)
    tup = O.as_numpy_tuples(t)
    p = workload("cfg2").preds[2]
    z = O.linear_logits(p, O.crop_features(p, F, tup["frame_id"], tup["bbox"]))
    ref = 7.0 * p["weight"].double().sum(1).numpy() + p["bias"].double().numpy()
    assert np.array_equal(z, np.tile(ref, (10, 1)))


def test_argmax_lowest_index_on_ties_and_margin():
    z = np.array([[1.0, 3.0, 3.0], [5.0, 5.0, 1.0], [0.0, -1.0, 2.0]])
    assert O.argmax_first(z).tolist() == [1, 0, 2]
    assert O.margin(z, 1).tolist() == [0.0, 0.0, -3.0]


def test_generator_makes_half_integer_target_margins():
    """R12 ("grid" heads): logits are multiples of s/2 (s = 2^-8) with the target at an odd multiple, so
    |margin| >= s/2 and fp32 accumulation is exact; and the workload's committed redraw table makes
    every margin of the covered tuples >= 0.05 (tests/oracle_cache.py)."""
    from synth.workload import WEIGHT_SCALE

    w = workload("cfg2", small=True)
    assert w.redraw is not None
    F = w.frames().numpy()
    t = w.tuples(n=300)
    tup = O.as_numpy_tuples(t)
    for p in w.preds[1:]:
        _, z = O.linear_verdict(p, F, tup["frame_id"], tup["bbox"], return_logits=True)
        m = O.margin(z, p["target"]) / WEIGHT_SCALE
        assert np.all(np.abs(m) >= 0.5) and np.all(np.abs(z / WEIGHT_SCALE) < 2 ** 22)
        assert np.all(np.mod(z[:, p["target"]] / WEIGHT_SCALE, 1.0) == 0.5)
        assert np.abs(O.margin(z, p["target"])).min() >= 0.05


def test_bf16_heads_redraw_table_guarantees_margins():
    """General bf16 heads (Q17): many weights are not fp16-representable, and with the committed redraw
    table every margin of the covered small-workload tuples is >= 0.05 (re-checked here with the
    oracle); redrawn tuples draw new bboxes, all other tuples are the plain generator's."""
    w = workload("cfg2", small=True, weights="bf16")
    plain = workload("cfg2", small=True, weights="bf16", redraw=False)
    ids, retry = w.redraw
    assert len(ids) > 0 and retry.min() >= 1
    F = w.frames().numpy()
    n = 2000
    t, t0 = w.tuples(n=n), plain.tuples(n=n)
    moved = ~(t.bbox == t0.bbox).all(dim=1).numpy()
    assert np.array_equal(np.where(moved)[0], ids[ids < n])
    tup = O.as_numpy_tuples(t)
    for p in w.preds[1:]:
        wf = p["weight"].float()
        assert (wf != wf.half().float()).float().mean() > 0.005
        _, z = O.linear_verdict(p, F, tup["frame_id"], tup["bbox"], return_logits=True)
        assert np.abs(O.margin(z, p["target"])).min() >= 0.05


# ----------------------------------------------------------------------------- MLP head (R25)


def _mlp_pred(W1, b1, W2, b2, target=0):
    return dict(kind="mlp", weight=torch.as_tensor(W1).to(torch.bfloat16), bias=torch.as_tensor(b1, dtype=torch.float32),
                weight2=torch.as_tensor(W2).to(torch.bfloat16), bias2=torch.as_tensor(b2, dtype=torch.float32),
                hidden=len(b1), n_classes=len(b2), target=target, crop_mode="nearest")


def test_mlp_one_hot_first_layer_selects_pixels():
    """W1 rows = e_{k_h}, b1 = 0 -> h = crop pixel x[k_h] (integers <= 255 are exact in bf16), so
    z = W2 x_sel + b2 with x from torch nearest-exact (a closed form through the whole head)."""
    F = make_frames(7, 2, 96, 128).numpy()
    t = make_tuples(7, 0, 30, n_frames=2, frame_h=96, frame_w=128, w_min=8, n_octaves=4)
    tup = O.as_numpy_tuples(t)
    picks = [(0, 0, 0), (5, 9, 1), (63, 63, 2), (40, 2, 0)]
    W1 = np.zeros((len(picks), O.K_FEATURES), np.float32)
    for h, (dy, dx, ch) in enumerate(picks):
        W1[h, (dy * 64 + dx) * 3 + ch] = 1.0
    W2 = np.array([[1.0, -2.0, 0.5, 0.0], [0.25, 0.0, 1.0, -1.0], [0.0, 0.0, 0.0, 0.0]], np.float32)
    b2 = np.array([0.5, -1.0, 3.0], np.float32)
    pred = _mlp_pred(W1, np.zeros(len(picks), np.float32), W2, b2)
    z = O.mlp_logits(pred, O.crop_features(pred, F, tup["frame_id"], tup["bbox"]))
    for i in range(len(tup["id"])):
        ref = torch.nn.functional.interpolate(_torch_crop(F[tup["frame_id"][i]], tup["bbox"][i]),
                                              size=(64, 64), mode="nearest-exact")[0]
        xs = np.array([float(ref[ch, dy, dx]) for (dy, dx, ch) in picks])
        assert np.allclose(z[i], W2.astype(np.float64) @ xs + b2, rtol=0, atol=1e-12)


def test_mlp_hidden_is_relu_then_bf16_round_to_nearest_even():
    """Single hidden unit a = x0 * w + b1 with hand-picked values: ReLU clips negatives, 257 ties to
    even (256), 258 is exact, 259 rounds up to 260 (bf16 has 8 significant bits)."""
    W1 = np.zeros((1, O.K_FEATURES), np.float32)
    W1[0, 0] = 1.0
    W2 = np.ones((1, 1), np.float32)
    for x0, b1, expect in [(10, -20.0, 0.0), (200, 57.0, 256.0), (200, 58.0, 258.0), (200, 59.0, 260.0),
                           (3, 0.25, 3.25)]:
        x = np.zeros((1, O.K_FEATURES))
        x[0, 0] = x0
        z = O.mlp_logits(_mlp_pred(W1, np.array([b1], np.float32), W2, np.zeros(1, np.float32)), x)
        assert z[0, 0] == expect, (x0, b1, z[0, 0], expect)


def test_mlp_matches_torch_bf16_pipeline_on_generated_head():
    """The generated head on real crops against torch's own ops (f64 matmul, relu, .to(bfloat16))."""
    w = workload("mlp", small=True)
    p = w.preds[1]
    F = w.frames().numpy()
    tup = O.as_numpy_tuples(w.tuples(n=64))
    x = O.crop_features(p, F, tup["frame_id"], tup["bbox"])
    xt = torch.from_numpy(x)
    a = xt @ p["weight"].double().T + p["bias"].double()
    h = torch.relu(a).to(torch.float32).to(torch.bfloat16).double()
    ref = h @ p["weight2"].double().T + p["bias2"].double()
    assert torch.allclose(torch.from_numpy(O.mlp_logits(p, x)), ref, rtol=0, atol=1e-9)
    # every hidden pre-activation of the generated head is s * integer (exact in fp32, R25)
    assert p["calib"]["weights"] == "grid"
    assert torch.all(torch.frac(a / WEIGHT_SCALE) == 0)


def test_mlp_all_negative_hidden_gives_bias_and_generated_selectivity():
    W1 = np.ones((2, O.K_FEATURES), np.float32)
    pred = _mlp_pred(W1, np.array([-1e9, -1e9], np.float32), np.ones((3, 2), np.float32),
                     np.array([1.0, 2.0, 3.0], np.float32), target=2)
    z = O.mlp_logits(pred, np.full((4, O.K_FEATURES), 255.0))
    assert np.array_equal(z, np.tile([1.0, 2.0, 3.0], (4, 1)))
    w = workload("mlp", small=True)
    tup = O.as_numpy_tuples(w.tuples(n=3000))
    v = O.linear_verdict(w.preds[1], w.frames().numpy(), tup["frame_id"], tup["bbox"])
    assert abs(v.mean() - 0.254) < 0.04


# ----------------------------------------------------------------------------- HSV colour heuristic (f4, R27)


def _all_rgb():
    v = np.arange(1 << 24, dtype=np.int64)
    return np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], axis=-1)


def test_rgb_to_hsv_equals_opencv_on_every_colour():
    """R27 reads DogColorClassifier's HSV as OpenCV's 8-bit cvtColor: the oracle's
    fixed-point steps equal cv2.cvtColor(COLOR_RGB2HSV) bit for bit on all 2^24 RGB colours, and so
    does the resulting colour class."""
    cv2 = pytest.importorskip("cv2")
    rgb = _all_rgb()
    ref = cv2.cvtColor(rgb.astype(np.uint8).reshape(4096, 4096, 3), cv2.COLOR_RGB2HSV).reshape(-1, 3)
    got = O.rgb_to_hsv_u8(rgb)
    assert np.array_equal(got, ref.astype(np.int64))
    assert np.array_equal(O.hsv_class(got), O.hsv_class(ref.astype(np.int64)))


def test_rgb_to_hsv_near_colorsys():
    """Against Python's colorsys (float HSV): V exact, S and H within one unit of 255 s / 180 h
    (the fixed-point reciprocals round once more than the float formula), and exact on the
    primaries, the secondaries and greys."""
    import colorsys

    rng = np.random.default_rng(11)
    rgb = rng.integers(0, 256, size=(20000, 3))
    got = O.rgb_to_hsv_u8(rgb)
    for (r, g, b), (H, S, V) in zip(rgb.tolist(), got.tolist()):
        h, s_, v = colorsys.rgb_to_hsv(r / 255, g / 255, b / 255)
        assert V == round(v * 255)
        assert abs(S - s_ * 255) <= 1.0
        dh = abs(H - h * 180)
        assert min(dh, 180 - dh) <= 1.0, ((r, g, b), H, h * 180)
    fixed = {(255, 0, 0): (0, 255, 255), (0, 255, 0): (60, 255, 255), (0, 0, 255): (120, 255, 255),
             (255, 255, 0): (30, 255, 255), (0, 255, 255): (90, 255, 255), (255, 0, 255): (150, 255, 255),
             (0, 0, 0): (0, 0, 0), (128, 128, 128): (0, 0, 128), (255, 255, 255): (0, 0, 255)}
    for k, v in fixed.items():
        assert tuple(O.rgb_to_hsv_u8(np.array(k)).tolist()) == v


def test_hsv_boxes_disjoint_over_all_colours_and_paper_red():
    """Every 8-bit RGB colour falls in at most one class box (so 'first box' = 'the box'), and the
    paper's red range (0, 50, 70)-(9, 255, 255) classifies as red."""
    hsv = O.rgb_to_hsv_u8(_all_rgb())
    hits = np.zeros(len(hsv), dtype=np.int64)
    for boxes in O.HSV_BOXES:
        inside = np.zeros(len(hsv), dtype=bool)
        for lo, hi in boxes:
            inside |= np.all((hsv >= np.array(lo)) & (hsv <= np.array(hi)), axis=-1)
        hits += inside
    assert hits.max() == 1
    assert O.hsv_class(np.array([[0, 50, 70], [9, 255, 255], [5, 200, 200]])).tolist() == [0, 0, 0]
    assert O.hsv_class(np.array([[10, 200, 200], [0, 49, 200], [0, 200, 69]])).tolist() == [9, 9, 9]


def test_hsv_counts_and_verdict_closed_forms():
    """A crop of a constant-colour frame has all 4096 pixels in that colour's class; ties in the
    counts go to the lowest class index."""
    for rgb, cls in [((200, 30, 30), 0), ((15, 15, 15), 1), ((40, 60, 200), 5), ((240, 240, 240), 8),
                     ((200, 120, 40), 9)]:
        F = np.zeros((1, 96, 128, 3), np.uint8)
        F[:] = rgb
        t = make_tuples(4, 0, 5, n_frames=1, frame_h=96, frame_w=128, w_min=8)
        tup = O.as_numpy_tuples(t)
        v, c = O.hsv_verdict(dict(kind="hsv", target=cls), F, tup["frame_id"], tup["bbox"], return_counts=True)
        assert np.all(c[:, cls] == 4096) and np.all(c.sum(1) == 4096) and v.all()
    assert O.argmax_first(np.array([[3.0, 5.0, 5.0, 1.0]])).tolist() == [1]


# ----------------------------------------------------------------------------- reuse-aware routing (f2)


def test_reuse_paper_example_orders_by_cached_range():
    """UC2: inside (1000, 7000) ObjectDetector's results are cached, so it goes
    first; inside (8000, 14000) HardHatDetector goes first; equal costs elsewhere keep the id order."""
    from synth import UC2_CACHED

    c = [64.0, 64.0]
    for lo, expect in [(2000, [0, 1]), (9000, [1, 0]), (0, [0, 1]), (14500, [0, 1]), (7200, [0, 1])]:
        ids = np.arange(lo, lo + 500)
        hits = [O.cache_hit_rate(ids, UC2_CACHED[k]) for k in range(2)]
        assert O.reuse_order(c, hits) == expect, (lo, hits)
    # a batch straddling the (8000, 14000) boundary: 60% cached -> estimated 0.4 * 64 < 64
    ids = np.arange(7600, 8601)
    hits = [O.cache_hit_rate(ids, UC2_CACHED[k]) for k in range(2)]
    assert abs(hits[1] - 600 / 1001) < 1e-12 and O.reuse_order(c, hits) == [1, 0]


def test_reuse_estimated_cost_equals_realized_compute_cost():
    """(1 - hit) * c is the compute cost per tuple when every uncached tuple costs c and cache hits
    cost nothing: brute-force count over random batches and cached ranges."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        ids = rng.integers(0, 10_000, size=rng.integers(1, 400))
        lo = int(rng.integers(0, 9000))
        cached = [(lo, lo + int(rng.integers(1, 3000)))]
        c = float(rng.uniform(0.1, 100))
        realized = sum(c for v in ids if not (cached[0][0] < v < cached[0][1])) / len(ids)
        assert abs(O.reuse_estimated_cost(c, O.cache_hit_rate(ids, cached)) - realized) < 1e-9 * c


def test_reuse_order_minimises_compute_cost_for_equal_selectivity():
    """With equal selectivities (so the order does not change which tuples reach the second
    predicate) the lowest-estimated-cost-first order minimises the expected compute cost
    e_1 + s * e_2 (brute force over both orders, E of R20 with estimated costs)."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        c = rng.uniform(1, 50, size=2)
        h = rng.uniform(0, 1, size=2)
        s = float(rng.uniform(0.05, 0.95))
        e = [O.reuse_estimated_cost(c[k], h[k]) for k in range(2)]
        best = min(itertools.permutations(range(2)), key=lambda p: O.expected_cost(p, e, [s, s]))
        assert O.expected_cost(O.reuse_order(c, h), e, [s, s]) <= O.expected_cost(best, e, [s, s]) + 1e-12


# ----------------------------------------------------------------------------- AND / order

def test_and_is_order_independent_brute_force():
    rng = np.random.default_rng(1)
    V = rng.random((4, 500)) < np.array([[0.3], [0.6], [0.9], [0.5]])
    ref = V.all(0)
    for perm in itertools.permutations(range(4)):
        n_in, n_pass, alive = O.sequential_eval(V, perm)
        assert np.array_equal(alive, ref)
        assert n_in[perm[0]] == 500 and n_pass[perm[-1]] == ref.sum()


def test_and_order_independent_on_real_predicates():
    w = workload("cfg2", small=True)
    F = w.frames().numpy()
    t = w.tuples(n=400)
    V = O.evaluate_all(w.preds, t, F)
    ids, _, keep = O.query_result(t, V)
    for perm in itertools.permutations(range(3)):
        assert np.array_equal(O.sequential_eval(V, perm)[2], keep)
    # n = 1 reduces to a plain filter
    assert np.array_equal(O.sequential_eval(V[:1], [0])[2], V[0])


# ----------------------------------------------------------------------------- rank / E / fold

def test_paper_score_example():
    g = GOLD["routing_example"]
    sb = O.score(g["breed"]["cost"], g["breed"]["selectivity"])
    sc = O.score(g["colour"]["cost"], g["colour"]["selectivity"])
    assert sb == pytest.approx(g["score_breed"]) and sc == pytest.approx(g["score_colour"]) and sb < sc


def test_paper_uc1_first_choice_per_policy():
    g = GOLD["uc1"]
    names = ["breed", "colour"]
    c = [g["breed"]["cost"], g["colour"]["cost"]]
    s = [g["breed"]["selectivity"], g["colour"]["selectivity"]]
    for pol, first in g["first_under"].items():
        keys = [O.policy_key(pol, ci, si) for ci, si in zip(c, s)]
        assert names[O.order_by_key(keys)[0]] == first


@pytest.mark.parametrize("case", ["case1", "case2"])
def test_paper_table1_colour_first(case):
    g = GOLD["table1"][case]
    c = [g["breed"]["cost"], g["colour"]["cost"]]
    s = [g["breed"]["selectivity"], g["colour"]["selectivity"]]
    for pol in ("score", "cost"):
        assert O.order_by_key([O.policy_key(pol, ci, si) for ci, si in zip(c, s)])[0] == 1


def test_sequential_timeline_closed_form():
    """Sequential (one resource) variant of PAPER.md:349-359: breed-first 2+0.1*1 = 2.1/item -> 21
    units for 10 items < colour-first 1+0.6*2 = 2.2 -> 22: the score order is optimal."""
    g = GOLD["routing_example"]
    c = [g["breed"]["cost"], g["colour"]["cost"]]
    s = [g["breed"]["selectivity"], g["colour"]["selectivity"]]
    assert O.expected_cost([0, 1], c, s) * g["items"] == pytest.approx(21.0)
    assert O.expected_cost([1, 0], c, s) * g["items"] == pytest.approx(22.0)
    assert O.order_by_key([O.score(ci, si) for ci, si in zip(c, s)]) == [0, 1]


def test_expected_cost_equals_enumeration_over_outcomes():
    """E(pi) vs exact enumeration over all 2**n independent verdict vectors (brute force)."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        n = int(rng.integers(1, 6))
        c, s = rng.random(n) * 10, rng.random(n)
        order = list(rng.permutation(n))
        tot = 0.0
        for bits in itertools.product([0, 1], repeat=n):
            pr = np.prod([s[k] if bits[k] else 1 - s[k] for k in range(n)])
            cost = 0.0
            for k in order:
                cost += c[k]
                if not bits[k]:
                    break
            tot += pr * cost
        assert O.expected_cost(order, c, s) == pytest.approx(tot, rel=1e-12)


def test_score_order_minimises_expected_cost_brute_force():
    """Hellerstein: sorting by c/(1-s) attains min_pi E(pi)."""
    rng = np.random.default_rng(3)
    for _ in range(2000):
        n = int(rng.integers(1, 7))
        c = rng.random(n) * 10
        s = rng.random(n) * 0.999
        best, _ = O.brute_force_best_orders(c, s)
        order = O.order_by_key([O.score(ci, si) for ci, si in zip(c, s)])
        assert O.expected_cost(order, c, s) <= best * (1 + 1e-12) + 1e-12


def test_score_special_cases():
    assert O.score(0.0, 0.7) == 0.0
    assert O.score(0.0, 1.0) == 0.0
    assert O.score(3.0, 1.0) == math.inf
    assert O.score(5.0, 0.0) == 5.0
    assert O.order_by_key([1.0, 1.0, 0.5]) == [2, 0, 1]  # ties -> lowest id


def test_fold_gamma_one_is_plain_counts_and_priors():
    f = O.FoldState(2, 1.0, declared_cost=[3.0, 7.0])
    assert f.sel() == [0.5, 0.5] and f.cost() == [3.0, 7.0]
    f.fold([1000, 0], [254, 0], [35110.0, 0.0])
    f.fold([1000, 0], [254, 0], [35110.0, 0.0])
    assert f.sel()[0] == pytest.approx(0.254) and f.cost()[0] == pytest.approx(35.11)
    assert f.sel()[1] == 0.5 and f.cost()[1] == 7.0  # unchanged when delta_in == 0
    g = O.FoldState(1, 0.5, declared_cost=[1.0])
    g.fold([100], [10], [100.0])
    g.fold([100], [90], [300.0])
    assert g.s_in == [150.0] and g.s_pass == [95.0] and g.s_cost == [350.0]


# ------------------------------------------------------------------ data-aware balance (f4, R28)

def _best_contiguous_max_load(chunk_cost, G):
    """Brute force: the smallest possible max load over all cuts of the chunks into G
    contiguous (possibly empty) ranges."""
    n = len(chunk_cost)
    best = None
    for cuts in itertools.combinations_with_replacement(range(n + 1), G - 1):
        b = (0,) + cuts + (n,)
        m = max(int(sum(chunk_cost[b[i]:b[i + 1]])) for i in range(G))
        best = m if best is None else min(best, m)
    return best


def test_balanced_bounds_load_bound_and_near_optimal_brute_force():
    """PAPER.md:863-882 balance the estimated loads: every worker's load is at most A/G plus one
    chunk, and the max load is within one chunk of the best contiguous cut (brute force)."""
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 8))
        G = int(rng.integers(1, 5))
        cc = rng.integers(0, 50, n).astype(np.int64)
        count = 32 * n - int(rng.integers(0, 32))
        b = O.balanced_bounds(cc, G, count)
        assert b[0] == 0 and b[-1] == count and all(b[i] <= b[i + 1] for i in range(G))
        assert all(x % 32 == 0 or x == count for x in b)
        loads = [int(cc[b[i] // 32:(b[i + 1] + 31) // 32].sum()) if b[i + 1] > b[i] else 0 for i in range(G)]
        A = int(cc.sum())
        assert sum(loads) == A
        assert max(loads) <= A / G + cc.max() + 1e-9
        assert max(loads) <= _best_contiguous_max_load(cc, G) + cc.max()


def test_balanced_bounds_uniform_cost_closed_form():
    """Equal chunk costs: worker c starts at chunk ceil(c * n / G) (closed form)."""
    for n in (1, 5, 37, 148, 1000):
        for G in (1, 3, 148):
            b = O.balanced_bounds(np.full(n, 7, np.int64), G, 32 * n)
            assert b == [min(32 * (-(-c * n // G)), 32 * n) for c in range(G)] + [32 * n]


def test_input_size_costs_and_loads_conserve_the_total():
    t = workload("cfg4", small=True, n=3000).tuples()
    tup = O.as_numpy_tuples(t)
    cost = O.input_size_costs(tup["bbox"])
    w = tup["bbox"][:, 2].astype(np.int64) - tup["bbox"][:, 0]
    h = tup["bbox"][:, 3].astype(np.int64) - tup["bbox"][:, 1]
    assert np.array_equal(cost, w * h)
    cc = O.chunk_costs(cost)
    assert int(cc.sum()) == int(cost.sum()) and len(cc) == (3000 + 31) // 32
    b = O.balanced_bounds(cc, 16, 3000)
    assert sum(O.range_loads(cost, b)) == int(cost.sum()) == sum(O.round_robin_loads(cost, 16))
    # on this heavy-tailed input size the data-aware cut beats round-robin's worst worker
    assert max(O.range_loads(cost, b)) < max(O.round_robin_loads(cost, 16))


# ------------------------------------------------------------- concurrent workers (f3, R29)

def _masks(n, k):
    for c in itertools.combinations(range(n), k):
        yield [i in c for i in range(n)]


def test_cost_route_timeline_paper_numbers():
    """PAPER.md:349-359 (Fig. cost_route): 10 items, DogColorClassifier cost 1 / selectivity 0.6,
    DogBreedClassifier cost 2 / selectivity 0.1, the two predicates on concurrent workers.
    Breed first: 20 time units (stage 1 is the bottleneck); colour first: 14 for the paper's
    arrival pattern, and 13..17 over every pattern of 6 passing items -- always below 20."""
    breed_first = [O.two_stage_completion(10, 2, 1, m) for m in _masks(10, 1)]
    assert breed_first[:-1] == [20.0] * 9 and breed_first[-1] == 21.0  # the last item passing adds its cost
    colour_first = [O.two_stage_completion(10, 1, 2, m) for m in _masks(10, 6)]
    assert O.two_stage_completion(10, 1, 2, [i + 1 in (2, 4, 6, 8, 9, 10) for i in range(10)]) == 14.0
    assert min(colour_first) == 13.0 and max(colour_first) == 17.0
    assert max(colour_first) < min(breed_first)
    # the routing decisions the paper derives: score picks breed (2/0.9 < 1/0.4), cost picks colour
    assert O.score(2, 0.1) < O.score(1, 0.6)


def test_fig7_cost_driven_never_worse_all_masks():
    """PAPER.md:548-556 (Fig. 7): A = 10 ms, B = 20 ms, sel_B in {0.1, 0.5, 0.9}, sel_A 0.1..0.9;
    cost-driven routing (A first) is never slower than selectivity- or score-driven routing:
    over every arrival pattern, A-first's worst completion <= the other order's best."""
    n = 10
    for sB in (0.1, 0.5, 0.9):
        for sA in [x / 10 for x in range(1, 10)]:
            kA, kB = round(sA * n), round(sB * n)
            a_first = [O.two_stage_completion(n, 10, 20, m) for m in _masks(n, kA)]
            b_first = [O.two_stage_completion(n, 20, 10, m) for m in _masks(n, kB)]
            assert max(a_first) <= min(b_first)


def test_flow_shop_closed_form_and_item_reduction():
    """Identical batches (a, b): makespan = a + b + (B - 1) * max(a, b) (closed form); one item per
    batch reduces the flow shop to the item timeline."""
    for a, b, B in ((1.0, 2.0, 10), (3.0, 1.0, 7), (2.5, 2.5, 4)):
        assert O.flow_shop_makespan([[a, b]] * B) == a + b + (B - 1) * max(a, b)
    rng = np.random.default_rng(3)
    for _ in range(50):
        m = rng.random(12) < 0.4
        rows = [[1.0, 2.0 if x else 0.0] for x in m]
        fs = O.flow_shop_makespan(rows)
        assert fs == O.two_stage_completion(12, 1.0, 2.0, m)


def test_pipeline_stage_times_counts_follow_eager_materialization():
    """Stage i of a batch is charged for exactly the tuples its predecessors passed (the counts of
    sequential_eval), times the worker's time per tuple."""
    rng = np.random.default_rng(5)
    V = rng.random((3, 1000)) < np.array([[0.6], [0.1], [0.5]])
    rows = O.pipeline_stage_times(V, [1, 0, 2], 250, [1.0, 2.0, 3.0])
    for b, row in enumerate(rows):
        n_in, _, _ = O.sequential_eval(V[:, 250 * b:250 * (b + 1)], [1, 0, 2])
        assert row == [n_in[1] * 2.0, n_in[0] * 1.0, n_in[2] * 3.0]


def test_area_division_by_reciprocal_is_correctly_rounded(tmp_path):
    """K4's AREA converter divides a bin sum by its pixel count as fma(fma(-q, b, a), y, q) with
    y = RN(1/b), q = RN(a*y) instead of an IEEE division; R10 needs RN(a/b).  The C program checks
    every integer a < 2^18 + 1 and count b <= 1100 (the largest AREA bin sum is 255 * 273)."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "check_area_div.c")
    exe = str(tmp_path / "check_area_div")
    subprocess.run([gcc, "-O2", "-mfma", "-ffp-contract=off", "-o", exe, src, "-lm"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip().startswith("bad 0 of"), r.stdout
