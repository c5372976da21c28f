"""Thin ctypes binding of libhydro's C ABI (include/hydro.h).

Argument marshalling only: every step of the eddy hot path runs in the library's CUDA
kernels.  torch is used for device memory (tensors whose data_ptr() is passed down) and
streams.  There is no CPU fallback: if libhydro.so is missing, importing this module's
functions raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# HYDRO_LIB_PATH selects an in-tree A/B variant (python -m paper_2403_14902_b200.build --variant ...)
LIB_PATH = os.environ.get("HYDRO_LIB_PATH") or os.path.join(HERE, "libhydro.so")

HYDRO_OK, HYDRO_EINVAL, HYDRO_ENOMEM, HYDRO_ECUDA, HYDRO_ENCCL, HYDRO_ESTATE, HYDRO_ERANGE, HYDRO_EBUSY = (
    0, -1, -2, -3, -4, -5, -6, -7)
BALANCE = {"round_robin": 0, "data_aware": 1}  # HYDRO_BALANCE_* (hydro.h)
POLICY = {"score": 0, "static": 1, "fixed": 2, "cost": 3, "selectivity": 4, "reuse": 5}
COST_SOURCE = {"measured": 0, "declared": 1}
PRED_KIND = {"label_eq": 0, "hash": 1, "linear": 2, "mlp": 3, "hsv": 4}
CROP_MODE = {"nearest": 0, "area": 1}
MAX_PRED = 8
FEATURES = 12288


class HydroError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hydro error {status}: {msg}")
        self.status = status


class hydro_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("policy", C.c_int32), ("cost_source", C.c_int32),
                ("decay_gamma", C.c_double), ("prior_selectivity", C.c_double), ("warmup_tuples", C.c_int64),
                ("max_batch_tuples", C.c_int64), ("max_inflight", C.c_int32), ("rank", C.c_int32),
                ("world", C.c_int32), ("sync_every", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("frames", C.c_void_p), ("n_frames", C.c_int32), ("frame_h", C.c_int32), ("frame_w", C.c_int32),
                ("balance", C.c_int32), ("max_sms", C.c_int32), ("sm_groups", C.c_int32), ("sm_group", C.c_int32),
                ("transport", C.c_int32), ("allreduce_fn", C.c_void_p), ("allreduce_user", C.c_void_p)]


# int32_t (*hydro_allreduce_fn)(void* user, uint64_t* data, int32_t count)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_uint64), C.c_int32)
TRANSPORT = {"nccl": 0, "host": 1}


class hydro_predicate_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("label_value", C.c_int32), ("seed", C.c_uint64),
                ("threshold", C.c_uint64 * 2), ("drift_id", C.c_uint64), ("units", C.c_int32),
                ("units_per_area", C.c_int32), ("weight_bf16", C.c_void_p), ("bias", C.c_void_p),
                ("weights_on_device", C.c_int32), ("n_classes", C.c_int32), ("target", C.c_int32),
                ("crop_mode", C.c_int32), ("hidden", C.c_int32), ("weight2_bf16", C.c_void_p), ("bias2", C.c_void_p),
                ("declared_cost", C.c_double), ("declared_selectivity", C.c_double)]


class hydro_tuples(C.Structure):
    _fields_ = [("id", C.c_void_p), ("frame_id", C.c_void_p), ("bbox", C.c_void_p), ("label", C.c_void_p),
                ("n", C.c_int64), ("on_device", C.c_int32), ("sel", C.c_void_p), ("sel_count", C.c_void_p),
                ("wait_event", C.c_void_p)]


class hydro_pred_stats(C.Structure):
    _fields_ = [("tuples_in", C.c_int64), ("tuples_passed", C.c_int64), ("cost_per_tuple", C.c_double),
                ("selectivity", C.c_double), ("rank", C.c_double), ("position", C.c_int32),
                ("s_in", C.c_double), ("s_pass", C.c_double), ("s_cost", C.c_double),
                ("cost_raw_total", C.c_double), ("tuples_computed", C.c_int64), ("cache_hit_rate", C.c_double),
                ("operand_fp16", C.c_int32), ("operand_scale_log2", C.c_int32), ("fused_pair", C.c_int32)]


class hydro_batch_report(C.Structure):
    _fields_ = [("n_tuples", C.c_int64), ("n_results", C.c_int64), ("warmup_tuples", C.c_int64),
                ("order_used", C.c_int32 * MAX_PRED), ("tuples_in", C.c_int64 * MAX_PRED),
                ("tuples_passed", C.c_int64 * MAX_PRED), ("cost_raw", C.c_double * MAX_PRED),
                ("tuples_computed", C.c_int64 * MAX_PRED), ("n_pred", C.c_int32)]


_P = C.c_void_p
_SIGS = {
    "hydro_version": ([], C.c_char_p),
    "hydro_last_error": ([], C.c_char_p),
    "hydro_config_default": ([C.POINTER(hydro_config)], C.c_int32),
    "hydro_nccl_unique_id": ([_P], C.c_int32),
    "hydro_create": ([C.POINTER(hydro_config), C.POINTER(_P)], C.c_int32),
    "hydro_add_predicate": ([_P, C.POINTER(hydro_predicate_desc), C.POINTER(C.c_int32)], C.c_int32),
    "hydro_set_fixed_order": ([_P, C.POINTER(C.c_int32), C.c_int32], C.c_int32),
    "hydro_cache_enable": ([_P, C.c_int32, C.c_uint64, C.c_int32], C.c_int32),
    "hydro_cache_put": ([_P, C.c_int32, _P, _P, C.c_int64, C.c_int32], C.c_int32),
    "hydro_cache_fill": ([_P, C.c_int32, C.POINTER(hydro_tuples)], C.c_int32),
    "hydro_submit_batch": ([_P, C.POINTER(hydro_tuples), C.POINTER(C.c_int64)], C.c_int32),
    "hydro_batch_count": ([_P, C.c_int64, C.POINTER(C.c_int64)], C.c_int32),
    "hydro_collect_results": ([_P, C.c_int64, _P, _P, C.c_int64, C.POINTER(C.c_int64), C.c_int32], C.c_int32),
    "hydro_release_batch": ([_P, C.c_int64], C.c_int32),
    "hydro_batch_output": ([_P, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)],
                           C.c_int32),
    "hydro_batch_info": ([_P, C.c_int64, C.POINTER(hydro_batch_report)], C.c_int32),
    "hydro_get_stats": ([_P, C.c_int32, C.POINTER(hydro_pred_stats)], C.c_int32),
    "hydro_get_order": ([_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int32),
    "hydro_synchronize": ([_P], C.c_int32),
    "hydro_flush_stats": ([_P], C.c_int32),
    "hydro_route_workers": ([C.POINTER(_P), C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                             C.POINTER(C.c_double)], C.c_int32),
    "hydro_launch_count": ([_P, C.POINTER(C.c_int64)], C.c_int32),
    "hydro_set_kernel_timing": ([_P, C.c_int32], C.c_int32),
    "hydro_kernel_time": ([_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int32),
    "hydro_device_time": ([_P, C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int32),
    "hydro_device_items": ([_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64)], C.c_int32),
    "hydro_debug_balance_bounds": ([_P, C.POINTER(C.c_uint32), C.c_int32, C.POINTER(C.c_int32)], C.c_int32),
    "hydro_destroy": ([_P], C.c_int32),
    "hydro_debug_linear": ([_P, C.c_int32, C.POINTER(hydro_tuples), _P, _P, _P], C.c_int32),
}
EXPORTS = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Loads libhydro.so (in-tree).  Raises if it is missing -- there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_2403_14902_b200.build`")
        _lib = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(_lib, name)
            f.argtypes = args
            f.restype = res
    return _lib


def _check(status: int):
    if status != HYDRO_OK:
        raise HydroError(status, lib().hydro_last_error().decode())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------------- C names

def hydro_version() -> str:
    return lib().hydro_version().decode()


def hydro_config_default() -> hydro_config:
    cfg = hydro_config()
    _check(lib().hydro_config_default(C.byref(cfg)))
    return cfg


def hydro_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().hydro_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def hydro_create(cfg: hydro_config) -> C.c_void_p:
    h = C.c_void_p()
    _check(lib().hydro_create(C.byref(cfg), C.byref(h)))
    return h


def hydro_add_predicate(ctx, desc: hydro_predicate_desc) -> int:
    pid = C.c_int32()
    _check(lib().hydro_add_predicate(ctx, C.byref(desc), C.byref(pid)))
    return pid.value


def hydro_cache_enable(ctx, pred_id: int, id_capacity: int, fill: bool = False):
    _check(lib().hydro_cache_enable(ctx, pred_id, id_capacity, 1 if fill else 0))


def hydro_cache_put(ctx, pred_id: int, ids, verdicts, on_device: bool):
    """ids: uint64-compatible (torch int64) 1-D, verdicts: uint8/bool 1-D, same length."""
    _check(lib().hydro_cache_put(ctx, pred_id, ids.data_ptr(), verdicts.data_ptr(), int(ids.numel()),
                                 1 if on_device else 0))


def hydro_cache_fill(ctx, pred_id: int, tup: hydro_tuples):
    _check(lib().hydro_cache_fill(ctx, pred_id, C.byref(tup)))


def hydro_set_fixed_order(ctx, order: Sequence[int]):
    arr = (C.c_int32 * len(order))(*order)
    _check(lib().hydro_set_fixed_order(ctx, arr, len(order)))


def hydro_submit_batch(ctx, tup: hydro_tuples) -> int:
    bid = C.c_int64()
    _check(lib().hydro_submit_batch(ctx, C.byref(tup), C.byref(bid)))
    return bid.value


def hydro_batch_count(ctx, batch_id: int) -> int:
    n = C.c_int64()
    _check(lib().hydro_batch_count(ctx, batch_id, C.byref(n)))
    return n.value


def hydro_collect_results(ctx, batch_id: int, ids_ptr, bbox_ptr, capacity: int, out_on_device: int) -> int:
    n = C.c_int64()
    _check(lib().hydro_collect_results(ctx, batch_id, ids_ptr, bbox_ptr, capacity, C.byref(n), out_on_device))
    return n.value


def hydro_release_batch(ctx, batch_id: int):
    _check(lib().hydro_release_batch(ctx, batch_id))


def hydro_batch_output(ctx, batch_id: int):
    """(positions, count, done_event) device pointers of an uncollected batch's survivors."""
    pos, cnt, ev = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _check(lib().hydro_batch_output(ctx, batch_id, C.byref(pos), C.byref(cnt), C.byref(ev)))
    return pos.value, cnt.value, ev.value


def hydro_batch_info(ctx, batch_id: int) -> hydro_batch_report:
    r = hydro_batch_report()
    _check(lib().hydro_batch_info(ctx, batch_id, C.byref(r)))
    return r


def hydro_get_stats(ctx, pred_id: int) -> hydro_pred_stats:
    s = hydro_pred_stats()
    _check(lib().hydro_get_stats(ctx, pred_id, C.byref(s)))
    return s


def hydro_get_order(ctx) -> List[int]:
    arr = (C.c_int32 * MAX_PRED)()
    n = C.c_int32()
    _check(lib().hydro_get_order(ctx, arr, C.byref(n)))
    return list(arr[: n.value])


def hydro_synchronize(ctx):
    _check(lib().hydro_synchronize(ctx))


def hydro_route_workers(ctxs: Sequence, policy: str):
    """(order, cost per tuple per worker, selectivity) from the workers' folded statistics (f3)."""
    n = len(ctxs)
    arr = (_P * n)(*[c.value if isinstance(c, C.c_void_p) else c for c in ctxs])
    order = (C.c_int32 * n)()
    cost = (C.c_double * n)()
    sel = (C.c_double * n)()
    _check(lib().hydro_route_workers(arr, n, POLICY[policy], order, cost, sel))
    return list(order), list(cost), list(sel)


def hydro_flush_stats(ctx):
    _check(lib().hydro_flush_stats(ctx))


def hydro_launch_count(ctx) -> int:
    n = C.c_int64()
    _check(lib().hydro_launch_count(ctx, C.byref(n)))
    return n.value


def hydro_set_kernel_timing(ctx, enable: bool):
    _check(lib().hydro_set_kernel_timing(ctx, 1 if enable else 0))


def hydro_kernel_time(ctx, kind: int):
    ms = C.c_double()
    n = C.c_int64()
    _check(lib().hydro_kernel_time(ctx, kind, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def hydro_device_time(ctx, kind: int, reset: bool = False):
    ms = C.c_double()
    n = C.c_int64()
    _check(lib().hydro_device_time(ctx, kind, 1 if reset else 0, C.byref(ms), C.byref(n)))
    return ms.value, n.value


def hydro_device_items(ctx, kind: int, reset: bool = False) -> int:
    n = C.c_int64()
    _check(lib().hydro_device_items(ctx, kind, 1 if reset else 0, C.byref(n)))
    return n.value


def hydro_debug_balance_bounds(ctx, capacity: int = 1024) -> List[int]:
    buf = (C.c_uint32 * capacity)()
    n = C.c_int32()
    _check(lib().hydro_debug_balance_bounds(ctx, buf, capacity, C.byref(n)))
    return list(buf[:n.value])


def hydro_destroy(ctx):
    _check(lib().hydro_destroy(ctx))


def hydro_debug_linear(ctx, pred_id: int, tup: hydro_tuples, logits=None, crops=None, verdict=None):
    _check(lib().hydro_debug_linear(ctx, pred_id, C.byref(tup), _ptr(logits), _ptr(crops), _ptr(verdict)))


# ---------------------------------------------------------------------------------- wrapper


def make_tuples_struct(id: torch.Tensor, frame_id: torch.Tensor, bbox: torch.Tensor, label: torch.Tensor):
    """SoA columns as torch tensors (int64 / int32 / int16[n,4] / int16, bit-compatible with u64/u32/u16)."""
    n = int(id.shape[0])
    for t, dt in ((id, torch.int64), (frame_id, torch.int32), (bbox, torch.int16), (label, torch.int16)):
        if t.dtype != dt or not t.is_contiguous():
            raise ValueError("tuple columns must be contiguous int64/int32/int16[n,4]/int16 tensors")
    on_dev = id.is_cuda
    if any(t.is_cuda != on_dev for t in (frame_id, bbox, label)):
        raise ValueError("tuple columns must all live on the same side")
    return hydro_tuples(id.data_ptr(), frame_id.data_ptr(), bbox.data_ptr(), label.data_ptr(), n, 1 if on_dev else 0)


class Eddy:
    """Convenience wrapper: one hydro context (one device, one stream)."""

    def __init__(self, *, device: int = 0, frames: Optional[torch.Tensor] = None, policy: str = "score",
                 cost_source: str = "measured", decay_gamma: float = 0.5, prior_selectivity: float = 0.5,
                 warmup_tuples: int = 65536, max_batch_tuples: int = 1 << 20, max_inflight: int = 4,
                 rank: int = 0, world: int = 1, sync_every: int = 1, nccl_unique_id: Optional[bytes] = None,
                 stream: Optional[torch.cuda.Stream] = None, balance: str = "round_robin", max_sms: int = 0,
                 sm_groups: int = 0, sm_group: int = 0, allreduce=None):
        """allreduce: HOST statistics transport (hydro.h HYDRO_TRANSPORT_HOST) -- a callable summing
        an int64 CPU tensor in place over the ranks, e.g. ``lambda t: dist.all_reduce(t)`` on a
        gloo group; None = NCCL (world > 1 needs nccl_unique_id)."""
        cfg = hydro_config_default()
        cfg.device = device
        cfg.stream = (stream or torch.cuda.current_stream(device)).cuda_stream
        cfg.policy = POLICY[policy]
        cfg.cost_source = COST_SOURCE[cost_source]
        cfg.decay_gamma = decay_gamma
        cfg.prior_selectivity = prior_selectivity
        cfg.warmup_tuples = warmup_tuples
        cfg.max_batch_tuples = max_batch_tuples
        cfg.max_inflight = max_inflight
        cfg.rank, cfg.world, cfg.sync_every = rank, world, sync_every
        cfg.balance = BALANCE[balance]
        cfg.max_sms = max_sms
        cfg.sm_groups, cfg.sm_group = sm_groups, sm_group
        self._uid = None
        self._allreduce = None
        if allreduce is not None:
            def _cb(user, data, count, _f=allreduce):
                try:
                    t = torch.frombuffer(C.cast(data, C.POINTER(C.c_uint8 * (8 * count))).contents,
                                         dtype=torch.int64)
                    _f(t)
                    return 0
                except Exception:  # reported as HYDRO_ENCCL by the library
                    return 1
            self._allreduce = ALLREDUCE_FN(_cb)  # kept alive for the context's lifetime
            cfg.transport = TRANSPORT["host"]
            cfg.allreduce_fn = C.cast(self._allreduce, C.c_void_p)
        if nccl_unique_id is not None:
            self._uid = C.create_string_buffer(nccl_unique_id, 128)
            cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        self.frames = frames
        if frames is not None:
            if frames.dtype != torch.uint8 or frames.dim() != 4 or frames.shape[3] != 3 or not frames.is_cuda:
                raise ValueError("frames must be a CUDA uint8 tensor [F, H, W, 3]")
            cfg.frames = frames.data_ptr()
            cfg.n_frames, cfg.frame_h, cfg.frame_w = int(frames.shape[0]), int(frames.shape[1]), int(frames.shape[2])
        self.cfg = cfg
        self.ctx = hydro_create(cfg)
        self.n_pred = 0
        self._keep: List[object] = []
        self._inflight: Dict[int, tuple] = {}  # batch id -> borrowed tensors (kept alive until collect)

    def add_predicate(self, p: Dict) -> int:
        d = hydro_predicate_desc()
        d.kind = PRED_KIND[p["kind"]]
        d.declared_cost = float(p.get("declared_cost", 1.0))
        d.declared_selectivity = float(p.get("declared_selectivity", 0.5))
        if p["kind"] == "label_eq":
            d.label_value = int(p["label"])
        elif p["kind"] == "hash":
            d.seed = int(p["seed"]) & (2 ** 64 - 1)
            d.threshold[0], d.threshold[1] = int(p["threshold"][0]), int(p["threshold"][1])
            d.drift_id = int(p["drift_id"])
            d.units = int(p.get("units", 1))
            d.units_per_area = int(p.get("units_per_area", 0))
        elif p["kind"] == "hsv":
            d.n_classes = 10
            d.target = int(p["target"])
            d.crop_mode = CROP_MODE[p.get("crop_mode", "nearest")]
        elif p["kind"] in ("linear", "mlp"):
            w = p["weight"].contiguous()
            b = p["bias"].to(torch.float32).contiguous()
            if w.dtype != torch.bfloat16 or w.shape[1] != FEATURES:
                raise ValueError("weight must be bf16 [rows, 12288]")
            w = w.view(torch.int16)
            d.weights_on_device = 1 if w.is_cuda else 0
            if b.is_cuda != w.is_cuda:
                b = b.to(w.device)
            self._keep += [w, b]
            d.weight_bf16 = w.data_ptr()
            d.bias = b.data_ptr()
            d.n_classes = int(p["n_classes"])
            d.target = int(p["target"])
            d.crop_mode = CROP_MODE[p.get("crop_mode", "nearest")]
            if p["kind"] == "mlp":
                w2 = p["weight2"].contiguous()
                b2 = p["bias2"].to(torch.float32).contiguous()
                if w2.dtype != torch.bfloat16 or w2.shape[1] != w.shape[0]:
                    raise ValueError("weight2 must be bf16 [C, hidden]")
                w2 = w2.view(torch.int16).to(w.device)
                b2 = b2.to(w.device)
                self._keep += [w2, b2]
                d.hidden = int(w.shape[0])
                d.weight2_bf16 = w2.data_ptr()
                d.bias2 = b2.data_ptr()
        pid = hydro_add_predicate(self.ctx, d)
        self.n_pred += 1
        return pid

    def set_fixed_order(self, order: Sequence[int]):
        hydro_set_fixed_order(self.ctx, list(order))

    def submit(self, tuples, sel=None, wait_event=None) -> int:
        """sel = (positions_ptr, count_ptr, capacity): device selection of the columns (R29)."""
        t = make_tuples_struct(tuples.id, tuples.frame_id, tuples.bbox, tuples.label)
        if sel is not None:
            t.sel, t.sel_count, t.n = sel[0], sel[1], int(sel[2])
        if wait_event is not None:
            t.wait_event = wait_event
        bid = hydro_submit_batch(self.ctx, t)
        # the C ABI borrows the columns until the batch is collected or released
        self._inflight[bid] = (tuples.id, tuples.frame_id, tuples.bbox, tuples.label)
        return bid

    def batch_output(self, batch_id: int):
        return hydro_batch_output(self.ctx, batch_id)

    def count(self, batch_id: int) -> int:
        return hydro_batch_count(self.ctx, batch_id)

    def collect(self, batch_id: int, device: str = "cpu", pin: bool = False):
        n = hydro_batch_count(self.ctx, batch_id)
        on_dev = device != "cpu"
        ids = torch.empty(max(n, 1), dtype=torch.int64, device=device, pin_memory=pin and not on_dev)
        bbox = torch.empty((max(n, 1), 4), dtype=torch.int16, device=device, pin_memory=pin and not on_dev)
        got = hydro_collect_results(self.ctx, batch_id, ids.data_ptr(), bbox.data_ptr(), n, 1 if on_dev else 0)
        self._inflight.pop(batch_id, None)
        return ids[:got], bbox[:got]

    def collect_into(self, batch_id: int, ids: torch.Tensor, bbox: torch.Tensor) -> int:
        """Copies the rows into caller buffers (host or device); returns the count."""
        got = hydro_collect_results(self.ctx, batch_id, ids.data_ptr(), bbox.data_ptr(), int(ids.shape[0]),
                                    1 if ids.is_cuda else 0)
        self._inflight.pop(batch_id, None)
        return got

    def release(self, batch_id: int):
        hydro_release_batch(self.ctx, batch_id)
        self._inflight.pop(batch_id, None)

    def flush_stats(self):
        """Multi-rank: fold every outstanding statistics window (collective over the ranks)."""
        hydro_flush_stats(self.ctx)

    def batch_info(self, batch_id: int) -> Dict:
        r = hydro_batch_info(self.ctx, batch_id)
        P = r.n_pred
        return dict(n_tuples=r.n_tuples, n_results=r.n_results, warmup_tuples=r.warmup_tuples,
                    order_used=list(r.order_used[:P]), tuples_in=list(r.tuples_in[:P]),
                    tuples_passed=list(r.tuples_passed[:P]), cost_raw=list(r.cost_raw[:P]),
                    tuples_computed=list(r.tuples_computed[:P]))

    def stats(self, pred_id: int) -> Dict:
        s = hydro_get_stats(self.ctx, pred_id)
        return {f: getattr(s, f) for f, _ in s._fields_}

    def order(self) -> List[int]:
        return hydro_get_order(self.ctx)

    def cache_enable(self, pred_id: int, id_capacity: int, fill: bool = False):
        hydro_cache_enable(self.ctx, pred_id, id_capacity, fill)

    def cache_fill(self, pred_id: int, tuples):
        """Evaluates pred_id alone on a device batch and caches its verdicts (UC2's Q1 / Q2)."""
        hydro_cache_fill(self.ctx, pred_id, make_tuples_struct(tuples.id, tuples.frame_id, tuples.bbox, tuples.label))

    def cache_put(self, pred_id: int, ids, verdicts):
        """Records verdicts of pred_id for tuple ids (torch tensors on the host or the GPU)."""
        v = verdicts.to(torch.uint8).contiguous()
        i = ids.to(torch.int64).contiguous()
        if i.is_cuda:
            v = v.to(i.device)
        hydro_cache_put(self.ctx, pred_id, i, v, i.is_cuda)
        if i.is_cuda:
            self.synchronize()  # device arrays are borrowed until the put ran

    def synchronize(self):
        hydro_synchronize(self.ctx)

    def launch_count(self) -> int:
        return hydro_launch_count(self.ctx)

    def set_kernel_timing(self, on: bool):
        hydro_set_kernel_timing(self.ctx, on)

    def kernel_time(self, kind: int):
        return hydro_kernel_time(self.ctx, kind)

    def device_time(self, kind: int, reset: bool = False):
        """(ms, launches) summed by the classifier kernels' device timers (kind 1 / 4 / 5)."""
        return hydro_device_time(self.ctx, kind, reset)

    def device_items(self, kind: int, reset: bool = False) -> int:
        """Classifier-input tuples (crops) the kind's launches evaluated, counted on the device."""
        return hydro_device_items(self.ctx, kind, reset)

    def debug_balance_bounds(self) -> List[int]:
        return hydro_debug_balance_bounds(self.ctx)

    def debug_linear(self, pred_id: int, tuples, logits=None, crops=None, verdict=None):
        t = make_tuples_struct(tuples.id, tuples.frame_id, tuples.bbox, tuples.label)
        hydro_debug_linear(self.ctx, pred_id, t, logits, crops, verdict)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            hydro_destroy(self.ctx)
            self.ctx = None
            self._inflight = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
