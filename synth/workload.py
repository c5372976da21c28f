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
* linear heads: weights 2^-8 * {-2..2} stored as bf16 (exact), biases 2^-8 * (integer, +1/2 on
  the target), so nearest-crop logits are exact multiples of 2^-9 and the target's margin is
  never 0 (reading R12);
* HASH predicates: threshold ``T = round(sel * 2**32)``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

GEN_VERSION = 1
M32 = 0xFFFFFFFF
_MULT = 0x45D9F3B  # < 2**27, so (x < 2**32) * _MULT < 2**59 fits int64

# stream ids
S_LABEL, S_LABEL2, S_WOCT, S_WOFF, S_HOCT, S_HOFF, S_X, S_Y, S_FRAME, S_WEIGHT = range(1, 11)
S_W1, S_W2 = 11, 12
S_BLOCK, S_NOISE = 13, 14
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
                device="cpu") -> Tuples:
    ids = torch.arange(id_start, id_start + n, dtype=torch.int64, device=device)
    frame_id = torch.div(ids, dets_per_frame, rounding_mode="floor") % n_frames
    dog_cut = int(round(p_dog * 2 ** 32))
    u = gen_u32(seed, S_LABEL, ids)
    other = gen_u32(seed, S_LABEL2, ids) % 79
    other = other + (other >= DOG_LABEL).to(torch.int64)
    label = torch.where(u < dog_cut, torch.full_like(u, DOG_LABEL), other)
    w = _octave_size(seed, S_WOCT, S_WOFF, ids, w_min, n_octaves, frame_w)
    h = _octave_size(seed, S_HOCT, S_HOFF, ids, w_min, n_octaves, frame_h)
    x0 = gen_u32(seed, S_X, ids) % (frame_w - w + 1)
    y0 = gen_u32(seed, S_Y, ids) % (frame_h - h + 1)
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


def make_linear_head(seed: int, n_classes: int, target: int, selectivity: float,
                     k_features: int = K_FEATURES):
    """Weights s * {-2..2} (s = 2^-8; exact in bf16 and fp16) and half-integer-offset biases.

    b_c = -s * floor(127.5 * sum_k W_ck) centres every logit; the target additionally
    gets s * (D + 0.5) with D = round(kappa * sigma) so that the (approximate, iid-Gaussian)
    pass rate is ``selectivity``.  Only the target bias carries the s/2, so with integer
    (nearest-crop) inputs every logit is an exact multiple of s/2 and the target never ties.
    """
    c = torch.arange(n_classes, dtype=torch.int64)[:, None]
    k = torch.arange(k_features, dtype=torch.int64)[None, :]
    wi = gen_u32(seed, S_WEIGHT, c * k_features + k) % 5 - 2
    rowsum = wi.sum(dim=1)
    bias = torch.floor(-127.5 * rowsum.to(torch.float64))
    sigma = math.sqrt(_PIX_VAR * float((wi * wi).sum(dim=1).to(torch.float64).mean()))
    kappa = target_offset_sigmas(n_classes, selectivity)
    bias[target] += round(kappa * sigma) + 0.5
    return ((wi.to(torch.float64) * WEIGHT_SCALE).to(torch.bfloat16), (bias * WEIGHT_SCALE).to(torch.float32),
            {"kappa": kappa, "sigma": sigma * WEIGHT_SCALE, "scale": WEIGHT_SCALE})


def make_mlp_head(seed: int, hidden: int, n_classes: int, target: int, selectivity: float,
                  k_features: int = K_FEATURES):
    """Two-layer head (R25): W1 = s*{-2..2} [hidden][K], b1 = -s*floor(127.5*rowsum)
    (centres every hidden pre-activation), W2 = s*{-2..2} [C][hidden], b2 centring the logits on
    the half-normal mean of the hidden units plus the target offset kappa*sigma_z (s = 2^-8).

    With integer (nearest-crop) inputs every hidden pre-activation is s * integer, exact in fp32,
    so its bf16 rounding is the same for any accumulation order.  Only the logits' f32 sums differ
    from float64 (tolerance 1e-2).  These are draws, not method arithmetic.
    """
    h = torch.arange(hidden, dtype=torch.int64)[:, None]
    k = torch.arange(k_features, dtype=torch.int64)[None, :]
    w1 = gen_u32(seed, S_W1, h * k_features + k) % 5 - 2
    b1 = torch.floor(-127.5 * w1.sum(dim=1).to(torch.float64))
    sigma1 = math.sqrt(_PIX_VAR * float((w1 * w1).sum(dim=1).to(torch.float64).mean())) * WEIGHT_SCALE
    c = torch.arange(n_classes, dtype=torch.int64)[:, None]
    hh = torch.arange(hidden, dtype=torch.int64)[None, :]
    w2 = gen_u32(seed, S_W2, c * hidden + hh) % 5 - 2
    w2f = w2.to(torch.float64) * WEIGHT_SCALE
    mean_h = sigma1 / math.sqrt(2.0 * math.pi)            # E[relu(N(0, sigma1))]
    var_h = sigma1 ** 2 * (0.5 - 1.0 / (2.0 * math.pi))   # Var[relu(N(0, sigma1))]
    sigma_z = math.sqrt(var_h * float((w2f * w2f).sum(dim=1).mean()))
    b2 = -mean_h * w2f.sum(dim=1)
    b2[target] += target_offset_sigmas(n_classes, selectivity) * sigma_z
    return ((w1.to(torch.float64) * WEIGHT_SCALE).to(torch.bfloat16), (b1 * WEIGHT_SCALE).to(torch.float32),
            w2f.to(torch.bfloat16), b2.to(torch.float32),
            {"sigma1": sigma1, "sigma_z": sigma_z, "scale": WEIGHT_SCALE})


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
                name=None):
    w, b, meta = make_linear_head(seed, n_classes, target, selectivity)
    return dict(kind="linear", weight=w, bias=b, target=target, n_classes=n_classes,
                crop_mode=crop_mode, declared_cost=declared_cost,
                declared_selectivity=float(selectivity), name=name or f"linear{n_classes}",
                calib=meta)


def make_color_frames(seed: int, n_frames: int, h: int, w: int, device="cpu", block: int = 16) -> torch.Tensor:
    """Frames of 16x16 blocks, each a palette colour (drawn per block) plus uniform noise in
    [-8, 8] per channel: crops cover a few blocks, so the HSV heuristic has a dominant colour."""
    f = torch.arange(n_frames, dtype=torch.int64, device=device)[:, None, None]
    y = torch.arange(h, dtype=torch.int64, device=device)[None, :, None]
    x = torch.arange(w, dtype=torch.int64, device=device)[None, None, :]
    blk = (f * ((h + block - 1) // block) + y // block) * ((w + block - 1) // block) + x // block
    pal = torch.tensor(PALETTE, dtype=torch.int64, device=device)
    base = pal[gen_u32(seed, S_BLOCK, blk) % len(PALETTE)]                      # [F, H, W, 3]
    pix = (f * h + y) * w + x
    ch = torch.arange(3, dtype=torch.int64, device=device)
    noise = gen_u32(seed, S_NOISE, pix[..., None] * 3 + ch) % 17 - 8
    return (base + noise).clamp(0, 255).to(torch.uint8)


def hsv_pred(target: int, selectivity: float, declared_cost=50.0, name=None):
    return dict(kind="hsv", target=target, n_classes=10, crop_mode="nearest", declared_cost=declared_cost,
                declared_selectivity=float(selectivity), name=name or f"hsv={target}")


def mlp_pred(seed, n_classes, target, selectivity, hidden=512, declared_cost=1000.0, name=None):
    w1, b1, w2, b2, meta = make_mlp_head(seed, hidden, n_classes, target, selectivity)
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

    def tuples(self, id_start=0, n=None, device="cpu") -> Tuples:
        return make_tuples(self.seed, id_start, self.n if n is None else n, n_frames=self.n_frames,
                           frame_h=self.frame_h, frame_w=self.frame_w, w_min=self.w_min,
                           n_octaves=self.n_octaves, device=device)

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


def workload(name: str, *, n: Optional[int] = None, small: bool = False) -> Workload:
    """BASELINE.json configs (cfg1..cfg5).  ``small`` shrinks frames for oracle-speed tests."""
    fh, fw, nf, wmin = (720, 1280, 1024, 32) if not small else (96, 128, 16, 8)
    if name == "cfg1":
        preds = [hash_pred(1, 0.5, units=1, name="A"), hash_pred(2, 0.1, units=10, name="B")]
        return Workload("cfg1", SEED, n or 10_000, 4, 96, 128, preds, policy="static", w_min=8,
                        batch_tuples=10_000, warmup_tuples=0,
                        notes="2 hash predicates sel 0.5/0.1 cost 1/10, static stats, one batch")
    if name == "cfg2":
        preds = [label_pred(),
                 linear_pred(SEED + 1, 120, 57, 0.254, name="breed=great dane"),
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black")]
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
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black"),
                 linear_pred(SEED + 1, 120, 57, 0.254, crop_mode="area", name="breed=great dane (area)")]
        return Workload("cfg4", SEED, n or 10_000_000, nf, fh, fw, preds, w_min=wmin,
                        batch_tuples=1 << 20,
                        notes="area-correlated classifier cost, 4 predicates")
    if name == "mlp":  # the dog query with the breed classifier as an MLP head
        preds = [label_pred(),
                 mlp_pred(SEED + 3, 120, 57, 0.254, name="breed=great dane (mlp)"),
                 linear_pred(SEED + 2, 10, 1, 0.633, name="colour=black")]
        return Workload("mlp", SEED, n or 1_000_000, nf, fh, fw, preds, w_min=wmin,
                        notes="cfg2 with a 12288-512-120 MLP breed head")
    if name == "hsv":  # the dog query with DogColorClassifier as the HSV heuristic
        preds = [label_pred(),
                 linear_pred(SEED + 1, 120, 57, 0.254, name="breed=great dane"),
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
        w = workload("cfg2", n=n or 100_000_000, small=small)
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
