"""Seeded synthetic workload generator (inputs only; no method arithmetic).

Everything is a pure function of ``(seed, stream, index)`` through a 32-bit
integer mixer (Mueller's ``hash32``; multiplier 0x45D9F3B).  It is written with
operators that behave identically on Python ints and on ``torch.int64`` tensors
(on CPU and on CUDA), and every intermediate product stays below 2**59, so the
same tuple / frame / weight is produced on any device.  This is deliberately a
DIFFERENT function from the method's HASH predicate (SplitMix64 + murmur3
fmix32, reading R5), so drawing inputs never computes a verdict.

Recipe (DESIGN.md §3 "Input recipe"):

* tuple ``id`` -> ``frame_id = (id // dets_per_frame) % n_frames`` (4 detections
  per frame, UNNEST of ObjectDetector(frame));
* ``label``: COCO id 16 ('dog') with probability ``p_dog``, else uniform over
  the other 79 classes;
* ``bbox``: half-open integer ``(x0, y0, x1, y1)``; width and height are drawn
  log-uniformly by octave in ``[w_min, w_min * 2**n_octaves)`` and clipped to
  the frame; the position is uniform inside the frame;
* frames: HWC uint8 noise, ``n_frames`` x H x W x 3;
* linear heads: ``weights="grid"``: 2^-8 * {-2..2} stored as bf16 (exact, also fp16-exact),
  biases 2^-8 * (integer, +1/2 on the target); ``weights="bf16"``: N(0, (2.5e-4)^2) rounded to
  bf16 (many are not fp16-representable), centring biases in f32;
* margin guarantee (R12): a tuple's bbox can be redrawn with a
  retry counter (``retry`` of ``make_tuples``: the draws use index ``id + retry * 2^40``); the
  counters come from a table written by ``tools/oracle_cache.py`` (which calls only ``oracle/``)
  so that every classifier margin of the workload is >= 0.05;
* HASH predicates: threshold ``T = round(sel * 2**32)``.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

GEN_VERSION = 2  # 2: per-tuple bbox redraw counters (margin guarantee, R12) and general bf16 heads
M32 = 0xFFFFFFFF
_MULT = 0x45D9F3B  # < 2**27, so (x < 2**32) * _MULT < 2**59 fits int64

# stream ids
S_LABEL, S_LABEL2, S_WOCT, S_WOFF, S_HOCT, S_HOFF, S_X, S_Y, S_FRAME, S_WEIGHT = range(1, 11)
S_W1, S_W2 = 11, 12
S_BLOCK, S_NOISE = 13, 14
S_GAUSS_A, S_GAUSS_B = 15, 16
REDRAW_STRIDE = 1 << 40  # draw index of a redrawn bbox: id + retry * 2^40 (ids < 2^40)
# palette of the coloured frame pool (RGB; one per HSV class of DESIGN.md R27, plus orange)
PALETTE = [(200, 30, 30), (15, 15, 15), (128, 128, 128), (220, 200, 40), (40, 160, 40), (40, 60, 200),
           (130, 40, 160), (230, 120, 170), (240, 240, 240), (200, 120, 40)]

CROP = 64
K_FEATURES = CROP * CROP * 3  # 12288
DOG_LABEL = 16  # COCO 'dog' (reading R15)


def mix32(x):
    """Mueller hash32 finaliser on values in [0, 2**32).  Works on ints and int64 tensors."""
    x = (((x >> 16) ^ x) * _MULT) & M32
    x = (((x >> 16) ^ x) * _MULT) & M32
    return (x >> 16) ^ x


def _stream_key(seed: int, stream: int) -> int:
    k = mix32(seed & M32) ^ ((seed >> 32) & M32)
    return mix32(k ^ mix32((stream * 0x9E3779B1) & M32))


def gen_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Counter-based draw: uniform u32 (as int64 in [0, 2**32)) for each non-negative idx."""
    k = _stream_key(seed, stream)
    h = mix32((idx & M32) ^ k)
    return mix32(h ^ (idx >> 32) ^ 0x6A09E667)


# ----------------------------------------------------------------------------------------------
# tuples


@dataclass
class Tuples:
    """Device- or host-resident SoA columns (torch tensors, bit-compatible with the C ABI)."""

    id: torch.Tensor        # int64  [n]   (u64 in the C ABI; ids < 2**63)
    frame_id: torch.Tensor  # int32  [n]   (u32)
    bbox: torch.Tensor      # int16  [n,4] (u16 x0,y0,x1,y1 half-open; values < 2**15)
    label: torch.Tensor     # int16  [n]   (u16)

    def __len__(self) -> int:
        return int(self.id.shape[0])

    def to(self, device, pin: bool = False) -> "Tuples":
        def mv(t):
            t = t.to(device)
            return t.pin_memory() if pin and t.device.type == "cpu" else t

        return Tuples(mv(self.id), mv(self.frame_id), mv(self.bbox), mv(self.label))

    def slice(self, a: int, b: int) -> "Tuples":
        return Tuples(self.id[a:b], self.frame_id[a:b], self.bbox[a:b], self.label[a:b])

    def select(self, idx) -> "Tuples":
        return Tuples(self.id[idx], self.frame_id[idx], self.bbox[idx], self.label[idx])

    def nbytes(self) -> int:
        return sum(int(t.numel() * t.element_size()) for t in (self.id, self.frame_id, self.bbox, self.label))


def _octave_size(seed, s_oct, s_off, ids, lo, n_oct, limit):
    octave = gen_u32(seed, s_oct, ids) % n_oct
    base = lo << octave  # lo * 2**octave
    v = base + gen_u32(seed, s_off, ids) % base
    return torch.clamp(v, max=limit)


def make_tuples(seed: int, id_start: int, n: int, *, n_frames: int, frame_h: int, frame_w: int,
                dets_per_frame: int = 4, p_dog: float = 0.5, w_min: int = 32, n_octaves: int = 3,
                device="cpu", retry: Optional[torch.Tensor] = None) -> Tuples:
    """``retry`` (int64 [n], optional): per-tuple bbox redraw counter (0 = the first draw)."""
    ids = torch.arange(id_start, id_start + n, dtype=torch.int64, device=device)
    frame_id = torch.div(ids, dets_per_frame, rounding_mode="floor") % n_frames
    dog_cut = int(round(p_dog * 2 ** 32))
    u = gen_u32(seed, S_LABEL, ids)
    other = gen_u32(seed, S_LABEL2, ids) % 79
    other = other + (other >= DOG_LABEL).to(torch.int64)
    label = torch.where(u < dog_cut, torch.full_like(u, DOG_LABEL), other)
    bidx = ids if retry is None else ids + retry.to(device=device, dtype=torch.int64) * REDRAW_STRIDE
    w = _octave_size(seed, S_WOCT, S_WOFF, bidx, w_min, n_octaves, frame_w)
    h = _octave_size(seed, S_HOCT, S_HOFF, bidx, w_min, n_octaves, frame_h)
    x0 = gen_u32(seed, S_X, bidx) % (frame_w - w + 1)
    y0 = gen_u32(seed, S_Y, bidx) % (frame_h - h + 1)
    bbox = torch.stack([x0, y0, x0 + w, y0 + h], dim=1)
    return Tuples(ids, frame_id.to(torch.int32), bbox.to(torch.int16), label.to(torch.int16))


# ----------------------------------------------------------------------------------------------
# frames


def make_frames(seed: int, n_frames: int, frame_h: int, frame_w: int, device="cpu",
                frame_ids: Optional[Sequence[int]] = None, out: Optional[torch.Tensor] = None,
                chunk_words: int = 1 << 24) -> torch.Tensor:
    """HWC uint8 noise frames. ``frame_ids`` selects a subset (id-addressable regeneration)."""
    if (frame_w * 3) % 4:
        raise ValueError("frame_w*3 must be a multiple of 4")
    wpf = frame_h * frame_w * 3 // 4
    fids = list(range(n_frames)) if frame_ids is None else [int(f) for f in frame_ids]
    if out is None:
        out = torch.empty((len(fids), frame_h, frame_w, 3), dtype=torch.uint8, device=device)
    flat = out.view(len(fids), -1)
    per = max(1, chunk_words // wpf)
    j = torch.arange(wpf, dtype=torch.int64, device=device)
    for a in range(0, len(fids), per):
        sel = fids[a:a + per]
        f = torch.tensor(sel, dtype=torch.int64, device=device)
        idx = (f[:, None] * wpf + j[None, :]).reshape(-1)
        v = gen_u32(seed, S_FRAME, idx)
        v = torch.where(v >= 2 ** 31, v - 2 ** 32, v).to(torch.int32)
        flat[a:a + len(sel)] = v.view(torch.uint8).view(len(sel), -1)
    return out


# ----------------------------------------------------------------------------------------------
# predicate parameters


def hash_threshold(sel: float) -> int:
    """T = round(sel * 2**32) in [0, 2**32] (reading R5)."""
    return int(min(max(round(sel * 2 ** 32), 0), 2 ** 32))


_PIX_VAR = (256.0 ** 2 - 1.0) / 12.0  # variance of a uniform u8


def _win_probability(kappa: float, n_classes: int) -> float:
    from scipy.special import ndtr

    u = np.linspace(-12.0, 12.0, 8001)
    phi = np.exp(-0.5 * u * u) / math.sqrt(2 * math.pi)
    return float(np.trapezoid(phi * ndtr(u + kappa) ** (n_classes - 1), u))


def target_offset_sigmas(n_classes: int, selectivity: float) -> float:
    """kappa with P(N(kappa,1) > max of C-1 iid N(0,1)) = selectivity (input calibration only)."""
    lo, hi = -12.0, 12.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if _win_probability(mid, n_classes) < selectivity:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


WEIGHT_SCALE = 2.0 ** -8  # keeps AREA-crop logits (non-integer inputs) well inside fp32 (R12)
BF16_SIGMA = 2.5e-4       # general bf16 heads: W ~ N(0, sigma^2)
BF16_W2_SIGMA = 0.03      # general bf16 MLP heads: second layer W2 ~ N(0, sigma^2)


def gen_normal(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Counter-based N(0, 1) draw (Box-Muller on two u32 draws), float64 on the CPU."""
    u1 = (gen_u32(seed, stream, idx).to(torch.float64) + 0.5) / 2.0 ** 32
    u2 = gen_u32(seed, stream + 100, idx).to(torch.float64) / 2.0 ** 32
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def _draw_weights(seed: int, stream: int, rows: int, cols: int, weights: str, sigma: float) -> torch.Tensor:
    """[rows][cols] float64 weights holding bf16 values: "grid" = s * {-2..2} (s = 2^-8),
    "bf16" = bf16(sigma * N(0, 1))."""
    r = torch.arange(rows, dtype=torch.int64)[:, None]
    c = torch.arange(cols, dtype=torch.int64)[None, :]
    idx = r * cols + c
    if weights == "grid":
        return (gen_u32(seed, stream, idx) % 5 - 2).to(torch.float64) * WEIGHT_SCALE
    if weights == "bf16":
        return (gen_normal(seed, stream, idx) * sigma).to(torch.bfloat16).to(torch.float64)
    raise ValueError(f"weights must be 'grid' or 'bf16', not {weights!r}")


def make_linear_head(seed: int, n_classes: int, target: int, selectivity: float,
                     k_features: int = K_FEATURES, weights: str = "grid"):
    """weights="grid": W = s * {-2..2} (s = 2^-8; exact in bf16 and fp16) and half-integer-offset
    biases: b_c = -s * floor(127.5 * sum_k W_ck / s) centres every logit; the target additionally
    gets s * (D + 0.5) with D = round(kappa * sigma / s) so that the (approximate, iid-Gaussian)
    pass rate is ``selectivity``.  weights="bf16": W = bf16(N(0, 2.5e-4^2)), b_c = f32(-127.5 *
    sum_k W_ck), target + kappa * sigma.  sigma is the logit spread over uniform-noise pixels.
    """
    W = _draw_weights(seed, S_WEIGHT, n_classes, k_features, weights, BF16_SIGMA)
    sigma = math.sqrt(_PIX_VAR * float((W * W).sum(dim=1).mean()))
    kappa = target_offset_sigmas(n_classes, selectivity)
    if weights == "grid":
        wi = torch.round(W / WEIGHT_SCALE)
        bias = torch.floor(-127.5 * wi.sum(dim=1))
        bias[target] += round(kappa * sigma / WEIGHT_SCALE) + 0.5
        bias = bias * WEIGHT_SCALE
    else:
        bias = -127.5 * W.sum(dim=1)
        bias[target] += kappa * sigma
    return W.to(torch.bfloat16), bias.to(torch.float32), {"kappa": kappa, "sigma": sigma, "weights": weights}


def make_mlp_head(seed: int, hidden: int, n_classes: int, target: int, selectivity: float,
                  k_features: int = K_FEATURES, weights: str = "grid"):
    """Two-layer head (R25): W1 [hidden][K], b1 = -127.5 * rowsum(W1) (floored to the s
    grid for "grid") centres every hidden pre-activation; W2 [C][hidden]; b2 centres the logits on
    the half-normal mean of the hidden units plus the target offset kappa * sigma_z.
    "grid": W1, W2 = s * {-2..2} (s = 2^-8): with integer (nearest-crop) inputs every hidden
    pre-activation is s * integer, exact in fp32.  "bf16": W1 = bf16(N(0, 2.5e-4^2)),
    W2 = bf16(N(0, 0.03^2)).  These are draws, not method arithmetic.
    """
    W1 = _draw_weights(seed, S_W1, hidden, k_features, weights, BF16_SIGMA)
    if weights == "grid":
        b1 = torch.floor(-127.5 * torch.round(W1 / WEIGHT_SCALE).sum(dim=1)) * WEIGHT_SCALE
    else:
        b1 = -127.5 * W1.sum(dim=1)
    sigma1 = math.sqrt(_PIX_VAR * float((W1 * W1).sum(dim=1).mean()))
    # W2 scale for "bf16": a hidden unit whose fp32 pre-activation lands on the other side of a bf16
    # rounding boundary than the f64 one moves a logit by |W2| * ulp_bf16(h) ~ 0.03 * 2^-7 (R25)
    w2f = _draw_weights(seed, S_W2, n_classes, hidden, weights, BF16_W2_SIGMA)
    mean_h = sigma1 / math.sqrt(2.0 * math.pi)            # E[relu(N(0, sigma1))]
    var_h = sigma1 ** 2 * (0.5 - 1.0 / (2.0 * math.pi))   # Var[relu(N(0, sigma1))]
    sigma_z = math.sqrt(var_h * float((w2f * w2f).sum(dim=1).mean()))
    b2 = -mean_h * w2f.sum(dim=1)
    b2[target] += target_offset_sigmas(n_classes, selectivity) * sigma_z
    return (W1.to(torch.bfloat16), b1.to(torch.float32), w2f.to(torch.bfloat16), b2.to(torch.float32),
            {"sigma1": sigma1, "sigma_z": sigma_z, "weights": weights})


# ----------------------------------------------------------------------------------------------
# predicate / workload descriptions (plain data)


def label_pred(label=DOG_LABEL, declared_cost=0.05, declared_selectivity=0.5, name="label=dog"):
    return dict(kind="label_eq", label=label, declared_cost=declared_cost,
                declared_selectivity=declared_selectivity, name=name)


def hash_pred(seed, sel, units=1, sel_after=None, drift_id=None, units_per_area=0,
              declared_cost=None, name=None):
    t0 = hash_threshold(sel)
    t1 = hash_threshold(sel if sel_after is None else sel_after)
    return dict(kind="hash", seed=seed, threshold=(t0, t1),
                drift_id=(2 ** 63 - 1 if drift_id is None else drift_id), units=units,
                units_per_area=units_per_area,
                declared_cost=float(units if declared_cost is None else declared_cost),
                declared_selectivity=float(sel), name=name or f"hash{seed}")


def linear_pred(seed, n_classes, target, selectivity, crop_mode="nearest", declared_cost=100.0,
                name=None, weights="grid"):
    w, b, meta = make_linear_head(seed, n_classes, target, selectivity, weights=weights)
    return dict(kind="linear", weight=w, bias=b, target=target, n_classes=n_classes,
                crop_mode=crop_mode, declared_cost=declared_cost,
                declared_selectivity=float(selectivity), name=name or f"linear{n_classes}",
                calib=meta)


def make_color_frames(seed: int, n_frames: int, h: int, w: int, device="cpu", block: int = 16,
                      chunk_frames: int = 8) -> torch.Tensor:
    """Frames of 16x16 blocks, each a palette colour (drawn per block) plus uniform noise in
    [-8, 8] per channel: crops cover a few blocks, so the HSV heuristic has a dominant colour.
    Generated `chunk_frames` frames at a time (the int64 intermediates of a whole 720p pool would
    not fit in host memory); the values do not depend on the chunking."""
    out = torch.empty((n_frames, h, w, 3), dtype=torch.uint8, device=device)
    pal = torch.tensor(PALETTE, dtype=torch.int64, device=device)
    y = torch.arange(h, dtype=torch.int64, device=device)[None, :, None]
    x = torch.arange(w, dtype=torch.int64, device=device)[None, None, :]
    ch = torch.arange(3, dtype=torch.int64, device=device)
    for a in range(0, n_frames, chunk_frames):
        f = torch.arange(a, min(a + chunk_frames, n_frames), dtype=torch.int64, device=device)[:, None, None]
        blk = (f * ((h + block - 1) // block) + y // block) * ((w + block - 1) // block) + x // block
        base = pal[gen_u32(seed, S_BLOCK, blk) % len(PALETTE)]                      # [F, H, W, 3]
        pix = (f * h + y) * w + x
        noise = gen_u32(seed, S_NOISE, pix[..., None] * 3 + ch) % 17 - 8
        out[a:a + f.shape[0]] = (base + noise).clamp(0, 255).to(torch.uint8)
    return out


def hsv_pred(target: int, selectivity: float, declared_cost=50.0, name=None):
    return dict(kind="hsv", target=target, n_classes=10, crop_mode="nearest", declared_cost=declared_cost,
                declared_selectivity=float(selectivity), name=name or f"hsv={target}")


def mlp_pred(seed, n_classes, target, selectivity, hidden=512, declared_cost=1000.0, name=None, weights="grid"):
    w1, b1, w2, b2, meta = make_mlp_head(seed, hidden, n_classes, target, selectivity, weights=weights)
    return dict(kind="mlp", weight=w1, bias=b1, weight2=w2, bias2=b2, hidden=hidden, target=target,
                n_classes=n_classes, crop_mode="nearest", declared_cost=declared_cost,
                declared_selectivity=float(selectivity), name=name or f"mlp{hidden}x{n_classes}", calib=meta)


@dataclass
class Workload:
    name: str
    seed: int
    n: int
    n_frames: int
    frame_h: int
    frame_w: int
    preds: List[Dict]
    policy: str = "score"
    w_min: int = 32
    n_octaves: int = 3
    batch_tuples: int = 1 << 20
    warmup_tuples: int = 65536
    notes: str = ""
    frame_kind: str = "noise"  # "noise" (uniform u8) or "color" (palette blocks, make_color_frames)
    weights: str = "grid"      # classifier weights: "grid" (fp16-exact) or "bf16" (general bf16)
    small: bool = False
    # bbox redraw table (R12 margin guarantee): sorted ids and their retry counters
    redraw: Optional[tuple] = None

    @property
    def key(self) -> str:
        """Name of the workload's oracle cache / redraw table (tests/golden/cache/<key>.npz)."""
        return f"{self.name}-{self.weights}{'-small' if self.small else ''}-g{GEN_VERSION}"

    def retry_for(self, id_start: int, n: int) -> Optional[torch.Tensor]:
        if self.redraw is None or n == 0:
            return None
        ids, retry = self.redraw
        a, b = np.searchsorted(ids, [id_start, id_start + n])
        if a == b:
            return None
        out = torch.zeros(n, dtype=torch.int64)
        out[torch.from_numpy(ids[a:b] - id_start)] = torch.from_numpy(retry[a:b].astype(np.int64))
        return out

    def tuples(self, id_start=0, n=None, device="cpu") -> Tuples:
        n = self.n if n is None else n
        return make_tuples(self.seed, id_start, n, n_frames=self.n_frames,
                           frame_h=self.frame_h, frame_w=self.frame_w, w_min=self.w_min,
                           n_octaves=self.n_octaves, device=device, retry=self.retry_for(id_start, n))

    def tuples_at(self, ids: np.ndarray, device="cpu") -> Tuples:
        """The tuples with the given (sorted, unique) ids, e.g. the 1 % sample id % 100 == 0."""
        ids = np.asarray(ids, dtype=np.int64)
        if len(ids) == 0:
            return self.tuples(0, 0, device)
        full = self.tuples(int(ids[0]), int(ids[-1]) - int(ids[0]) + 1, device="cpu")
        return full.select(torch.from_numpy(ids - ids[0])).to(device)

    def frames(self, device="cpu", frame_ids=None) -> torch.Tensor:
        if self.frame_kind == "color":
            f = make_color_frames(self.seed, self.n_frames, self.frame_h, self.frame_w, device=device)
            return f if frame_ids is None else f[frame_ids]
        return make_frames(self.seed, self.n_frames, self.frame_h, self.frame_w, device=device,
                           frame_ids=frame_ids)

    @property
    def needs_frames(self) -> bool:
        return any(p["kind"] in ("linear", "mlp", "hsv") for p in self.preds)


SEED = 20240321
CACHE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "cache")


def load_redraw(key: str):
    """The bbox redraw table of a workload (written by tests/oracle_cache.py, which calls only
    oracle/), or None when there is none."""
    path = os.path.join(CACHE_DIR, key + ".npz")
    if not os.path.exists(path):
        return None
    with np.load(path) as z:
        return z["redraw_ids"].astype(np.int64), z["redraw_retry"].astype(np.int64)


def workload(name: str, *, n: Optional[int] = None, small: bool = False, weights: str = "grid",
             redraw: bool = True) -> Workload:
    """BASELINE.json configs (cfg1..cfg5).  ``small`` shrinks frames for oracle-speed tests;
    ``weights`` picks the classifier heads' weight draw ("grid" or "bf16"); ``redraw`` applies the
    workload's committed bbox redraw table (margin guarantee) when one exists."""
    w = _workload(name, n=n, small=small, weights=weights)
    w.weights, w.small = weights, small
    if redraw and any(p["kind"] in ("linear", "mlp") for p in w.preds):
        w.redraw = load_redraw(w.key)
    return w


def _workload(name: str, *, n: Optional[int], small: bool, weights: str) -> Workload:
    fh, fw, nf, wmin = (720, 1280, 1024, 32) if not small else (96, 128, 16, 8)
    W = weights
    if name == "cfg1":
        preds = [hash_pred(1, 0.5, units=1, name="A"), hash_pred(2, 0.1, units=10, name="B")]
        return Workload("cfg1", SEED, n or 10_000, 4, 96, 128, preds, policy="static", w_min=8,
                        batch_tuples=10_000, warmup_tuples=0,
                        notes="2 hash predicates sel 0.5/0.1 cost 1/10, static stats, one batch")
    if name == "cfg2":
        preds = [label_pred(),
                 linear_pred(SEED + 1, 120, 57, 0.254, name="breed=great dane", weights=W),
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black", weights=W)]
        return Workload("cfg2", SEED, n or 1_000_000, nf, fh, fw, preds, w_min=wmin,
                        batch_tuples=1 << 20,
                        notes="dog query: label='dog' AND breed AND colour, linear heads, 64x64 nearest crops")
    if name == "cfg3":
        half = (n or 1_000_000) // 2
        preds = [hash_pred(11, 0.9, units=2, sel_after=0.1, drift_id=half, name="P0"),
                 hash_pred(12, 0.5, units=4, sel_after=0.5, drift_id=half, name="P1"),
                 hash_pred(13, 0.1, units=8, sel_after=0.9, drift_id=half, name="P2")]
        return Workload("cfg3", SEED, n or 1_000_000, 4, 96, 128, preds, w_min=8,
                        batch_tuples=65536,
                        notes="3 hash predicates, selectivity drift at id n/2")
    if name == "cfg4":
        preds = [label_pred(),
                 hash_pred(21, 0.5, units=1, units_per_area=4096, name="hash(area)"),
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black", weights=W),
                 linear_pred(SEED + 1, 120, 57, 0.254, crop_mode="area", name="breed=great dane (area)", weights=W)]
        return Workload("cfg4", SEED, n or 10_000_000, nf, fh, fw, preds, w_min=wmin,
                        batch_tuples=1 << 20,
                        notes="area-correlated classifier cost, 4 predicates")
    if name == "mlp":  # the dog query with the breed classifier as an MLP head
        preds = [label_pred(),
                 mlp_pred(SEED + 3, 120, 57, 0.254, name="breed=great dane (mlp)", weights=W),
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black", weights=W)]
        return Workload("mlp", SEED, n or 1_000_000, nf, fh, fw, preds, w_min=wmin,
                        notes="cfg2 with a 12288-512-120 MLP breed head")
    if name == "hsv":  # the dog query with DogColorClassifier as the HSV heuristic
        preds = [label_pred(),
                 linear_pred(SEED + 1, 120, 57, 0.254, name="breed=great dane", weights=W),
                 hsv_pred(1, 0.1, name="colour=black (hsv)")]
        return Workload("hsv", SEED, n or 1_000_000, nf, fh, fw, preds, w_min=wmin, frame_kind="color",
                        notes="cfg2 with the HSV colour heuristic on a coloured-block frame pool")
    if name == "uc2":  # PAPER.md:562-605 reuse-aware routing, HASH stand-ins for the two detectors
        preds = [hash_pred(SEED + 11, 0.5, units=64, declared_cost=64.0, name="ObjectDetector 'person'"),
                 hash_pred(SEED + 12, 0.5, units=64, declared_cost=64.0, name="HardHatDetector 'no hardhat'")]
        return Workload("uc2", SEED, n or 15_000, 4, 96, 128, preds, policy="reuse", w_min=8,
                        batch_tuples=1000, warmup_tuples=0,
                        notes="verdicts cached for ids in (1000, 7000) (predicate 0) and (8000, 14000) (predicate 1)")
    if name == "cfg5":
        w = _workload("cfg2", n=n or 100_000_000, small=small, weights=weights)
        w.name = "cfg5"
        w.notes = "cfg2 query, 100M tuples sharded over ranks"
        return w
    raise KeyError(name)


UC2_CACHED = ([(1000, 7000)], [(8000, 14000)])  # per predicate, cached id ranges


def shard_range(n: int, rank: int, world: int):
    """Contiguous id range [a, b) of rank r: rank-ordered concatenation = input order."""
    a = (n * rank) // world
    b = (n * (rank + 1)) // world
    return a, b
