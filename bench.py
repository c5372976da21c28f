"""Benchmark: tuples/s through the 3-predicate UDF conjunction (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[1] / SURVEY.md §8 cfg2): 1M synthetic dog-query detections per
GPU per step -- label = 'dog' AND DogBreed(Crop) = 'great dane' AND DogColor(Crop) = 'black' with
linear heads on 64x64 nearest crops of a 1024-frame 720p HWC uint8 pool (PAPER.md:43-49,
276-288).  A step = one routing batch of 1M tuples through the whole eddy hot path (order,
label / classifier hops with eager compaction, emit of (id, bbox), fold).  N > 1: one process
per GPU (torchrun), contiguous per-rank id shards (weak scaling), NCCL all-reduce of the
statistics deltas inside libhydro.

value  : device-timed (CUDA events on the context stream), inputs resident in HBM.
e2e    : same metric through the C ABI with pinned HOST tuple columns (H2D inside the timed
         region) and results copied back to pinned host memory (D2H), host wall clock.
roofline: the classifier kernel (K4), HBM-bound: algorithmic bytes = (12288 sampled crop bytes
         + 16 B metadata) per classifier-input tuple, over the kernel's summed
         CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tuples/sec through 3-predicate UDF conjunction at 1/2/4/8 B200; % HBM/tensor roofline"
UNIT = "tuples/s"
TUPLES_PER_STEP = 1_000_000
ROTATING_BATCHES = 6          # 6 x 22 MB of tuple columns + 2.83 GB frames: inputs larger than L2
K4_FEATURES = 12288
K4_BYTES_PER_TUPLE = K4_FEATURES + 16
WORKLOAD = ("cfg2: 1M dog-query detections per GPU per step; label='dog' AND breed(C=120) AND "
            "colour(C=10) linear heads on 64x64 nearest crops; 1024 x 720x1280x3 u8 frame pool")
WORKLOAD_HSV = ("hsv (SURVEY.md §8(f) f4): cfg2 with DogColorClassifier as the paper's HSV heuristic on a "
                "coloured-block frame pool (1024 x 720x1280x3), breed linear C=120; 1M detections per GPU per step")
WORKLOAD_MLP = ("mlp (SURVEY.md §8(f) f1): cfg2 with the breed classifier as a 12288-512-120 MLP head "
                "(bf16 hidden), colour linear C=10; 1M detections per GPU per step; 1024 x 720x1280x3 frames")


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """SM clock + throttle reasons polled through NVML every 5 ms during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            self._stop.wait(0.005)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        nv = self.nv
        names = {"hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        reasons = sorted({n for _, rs in self.samples for n, bit in names.items() if rs & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def _profile_traffic(name: str):
    """bytes_per_launch of a committed ncu capture (profiles/<name>), only if it was captured on the
    current library sources (csrc_sha16 stamp); else (None, why)."""
    path = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(path):
        return None, "no capture"
    try:
        d = json.load(open(path))
    except Exception as ex:
        return None, f"unreadable: {ex}"
    if d.get("csrc_sha16") != csrc_sha16():
        return None, f"stale: profiles/{name} was captured on sources {d.get('csrc_sha16')}, not {csrc_sha16()}"
    return d.get("bytes_per_launch"), f"profiles/{name} ({d.get('source', 'ncu')}), same sources"


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


PAPER_CONTEXT = {"speedup": "up to 11.52x over the EvaDB baseline (UC3, long video, Eddy + Laminar on 2 GPUs)",
                 "hardware": "2 x NVIDIA A40 (48 GB) on an AMD EPYC 7452 32-core server, CUDA 12.0",
                 "cite": "PAPER.md:16, 383-385, 785 (§4.2 setup, §5.2 UC3)",
                 "note": "context only: another system, machine and workload"}


def csrc_sha16() -> str:
    """Hash of the library sources (csrc/*, include/hydro.h): stamps profile-derived numbers."""
    import hashlib

    from paper_2403_14902_b200 import build as B

    h = hashlib.sha256()
    for f in B.sources():
        h.update(os.path.basename(f).encode())
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


_ORC = {}


def _oracle_chunk(bounds):
    from threadpoolctl import threadpool_limits

    import oracle as O

    a, b = bounds
    with threadpool_limits(1):
        O.evaluate_all(_ORC["w"].preds, _ORC["t"].slice(a, b), _ORC["frames"])
    return b - a


def cpu_oracle_rate(w, tuples_cpu, frames_host, seconds: float = 15.0, chunk: int = 256):
    """The oracle as it stands (every predicate on every tuple, f64 numpy) on the host: first one
    thread (BLAS limited to 1) on one chunk, then every core -- one single-threaded worker process
    per core over consecutive chunks of the same sample -- for about `seconds`.  Returns both rates
    and the sample sizes; `cores` = the worker processes that ran."""
    import multiprocessing as mp

    _ORC.update(w=w, t=tuples_cpu, frames=frames_host)
    t0 = time.perf_counter()
    one = _oracle_chunk((0, chunk))
    r1 = one / (time.perf_counter() - t0)
    procs = os.cpu_count() or 1
    n_target = int(min(len(tuples_cpu), max(procs * chunk, r1 * procs * seconds)))
    spans = [(a, min(a + chunk, n_target)) for a in range(0, n_target, chunk)]
    with mp.get_context("fork").Pool(procs) as pool:
        t0 = time.perf_counter()
        done = sum(pool.map(_oracle_chunk, spans, chunksize=1))
        el = time.perf_counter() - t0
    return {"value": done / el, "cores": procs, "tuples": done, "seconds": el, "one_thread_value": r1,
            "one_thread_tuples": one, **cpu_info()}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host (rank 0 only), same metric/config."""
    world, rank, local = _dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle as O
    from synth import workload
    from threadpoolctl import threadpool_info

    import multiprocessing as mp

    w = workload("cfg2", weights=args.weights)
    procs = os.cpu_count() or 1
    per_step = 16 * procs  # one 16-tuple chunk per core per step: a bounded sample of the workload
    t = w.tuples(n=per_step * 4)
    fids = np.unique(t.frame_id.numpy())
    frames = np.zeros((w.n_frames, w.frame_h, w.frame_w, 3), np.uint8)
    frames[fids] = w.frames(frame_ids=fids).numpy()
    _ORC.update(w=w, t=t, frames=frames)
    cores = procs
    times = []
    with mp.get_context("fork").Pool(procs) as pool:
        for s in range(args.warmup + args.steps):
            a = (s % 4) * per_step
            t0 = time.perf_counter()
            pool.map(_oracle_chunk, [(a + 16 * i, a + 16 * (i + 1)) for i in range(procs)], chunksize=1)
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
    el = sum(times)
    value = per_step * len(times) / el
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * el / len(times),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": WORKLOAD, "weights": args.weights, "tuples_per_step": per_step,
                                           "parallelism": f"{procs} single-threaded oracle processes (one per host core)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", **cpu_info(),
                            "sample": f"{per_step} tuples per step of the cfg2 workload ({procs} chunks of 16 in "
                                      f"parallel), every predicate on every tuple"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def run_gpu(args):
    import numpy as np
    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from paper_2403_14902_b200.dist import broadcast_unique_id, max_over_ranks, shard_ids
    from synth import workload

    world, rank, local = _dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        B.build()
    if dist:
        dist.barrier()
    mlp = args.workload == "mlp"
    hsv = args.workload == "hsv"
    w = workload("mlp" if mlp else ("hsv" if hsv else "cfg2"), weights=args.weights)
    frames = w.frames(device="cuda")
    uid = broadcast_unique_id(dist, rank, H.hydro_nccl_unique_id) if world > 1 else None
    stream = torch.cuda.current_stream()
    e = H.Eddy(frames=frames, policy="score", warmup_tuples=65536, max_batch_tuples=1 << 20,
               max_inflight=4, rank=rank, world=world, sync_every=1, nccl_unique_id=uid, stream=stream)
    for p in w.preds:
        e.add_predicate(p)
    # per-rank contiguous shard of each step's id range (weak scaling: 1M tuples per GPU per step)
    batches = []
    for b in range(ROTATING_BATCHES):
        start, _ = shard_ids(TUPLES_PER_STEP, rank, world, b)
        batches.append(w.tuples(id_start=start, n=TUPLES_PER_STEP, device="cuda"))
    res_ids = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
    res_bb = torch.empty((1 << 20, 4), dtype=torch.int16, device="cuda")

    def collect_dev(bid):
        return e.collect_into(bid, res_ids, res_bb)

    def run_steps(k, offset):
        pend = []
        for s in range(k):
            pend.append(e.submit(batches[(offset + s) % ROTATING_BATCHES]))
            if len(pend) >= 3:
                collect_dev(pend.pop(0))
        for bid in pend:
            collect_dev(bid)

    lin = [k for k, p in enumerate(w.preds) if p["kind"] == "linear"]
    mlps = [k for k, p in enumerate(w.preds) if p["kind"] == "mlp"]
    hsvs = [k for k, p in enumerate(w.preds) if p["kind"] == "hsv"]

    def hsv_in():
        return sum(e.stats(k)["tuples_in"] for k in hsvs)

    def lin_in():
        return sum(e.stats(k)["tuples_in"] for k in lin)

    def mlp_in():
        return sum(e.stats(k)["tuples_in"] for k in mlps)

    run_steps(max(args.warmup, 3), 0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # classifier tuples in and the device launch timers, read around the timed region (outside it)
    in_t0, min_t0, hin_t0 = lin_in(), mlp_in(), hsv_in()
    for kind in (1, 4, 5):
        e.device_time(kind, reset=True)
        e.device_items(kind, reset=True)
    launches0 = e.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        run_steps(args.steps, 1)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = e.launch_count() - launches0
    if dist:
        ms = max_over_ranks(ms, dist, "cuda")
        dist.barrier()
    value = world * TUPLES_PER_STEP * args.steps / (ms / 1000.0)
    # ---- the classifier kernels' share of THIS timed run: device launch timers (%globaltimer of the
    # first CTA start / last CTA end of every launch that evaluated a hop; no host events)
    k4_ms, k4_n = e.device_time(1)
    km_ms, km_n = e.device_time(4)
    kh_ms, kh_n = e.device_time(5)
    k4_evals = lin_in() - in_t0  # head evaluations as a sequential eddy counts them (folded statistics)
    # crops K4 gathered in the timed run, counted by the kernels (a fused pair's crops once)
    k4_tuples = e.device_items(1)
    pair_ks = [k for k in lin if e.stats(k)["fused_pair"]]
    km_tuples = e.device_items(4)
    kh_tuples = e.device_items(5)
    op_fp16 = [e.stats(k)["operand_fp16"] for k in lin + mlps]
    op_scale = [e.stats(k)["operand_scale_log2"] for k in lin]
    # ---- breakdown of the rest of the step (separate pass, CUDA events around every launch)
    e.set_kernel_timing(True)
    run_steps(args.steps, 2)
    k1_ms, k1_n = e.kernel_time(0)
    k5_ms, k5_n = e.kernel_time(2)
    k2c_ms, k2c_n = e.kernel_time(3)
    e.set_kernel_timing(False)
    k4_bytes = k4_tuples * K4_BYTES_PER_TUPLE
    peaks = _peaks()
    achieved = k4_bytes / (k4_ms / 1000.0) / 1e9 if k4_ms > 0 else 0.0
    traffic, traffic_note = _profile_traffic("k4_dram_traffic.json")

    # ---- e2e through the C ABI with pinned host buffers
    depth = args.e2e_depth  # batches in flight (2: measured no worse than 3, less noisy)
    host_batches = [batches[b].to("cpu", pin=True) for b in range(depth)]
    out_ids = torch.empty(1 << 20, dtype=torch.int64).pin_memory()
    out_bb = torch.empty((1 << 20, 4), dtype=torch.int16).pin_memory()
    h2d = host_batches[0].nbytes()
    d2h = []

    def e2e_steps(k):
        pend = []
        for s in range(k):
            pend.append(e.submit(host_batches[s % depth]))
            if len(pend) >= depth:
                n = e.collect_into(pend.pop(0), out_ids, out_bb)
                d2h.append(16 * n)
        for bid in pend:
            n = e.collect_into(bid, out_ids, out_bb)
            d2h.append(16 * n)

    e2e_steps(2)
    d2h.clear()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_steps(args.steps)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if dist:
        el = max_over_ranks(el, dist, "cuda")
    e2e_value = world * TUPLES_PER_STEP * args.steps / el

    order = e.order()
    sel = {w.preds[k]["name"]: round(e.stats(k)["selectivity"], 4) for k in range(len(w.preds))}
    cost = {w.preds[k]["name"]: round(e.stats(k)["cost_per_tuple"], 2) for k in range(len(w.preds))}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fr_host = frames.cpu().numpy()
        tc = batches[0].to("cpu")
        r = cpu_oracle_rate(w, tc, fr_host, seconds=args.cpu_seconds)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
               "nproc": r["nproc"], "cpu_model": r["cpu_model"],
               "one_thread": {"value": r["one_thread_value"], "tuples": r["one_thread_tuples"]},
               "sample": f"first {r['tuples']} tuples of the step's 1M-tuple batch ({r['seconds']:.1f} s wall on "
                         f"{r['cores']} single-threaded oracle processes), every predicate on every tuple, f64 numpy"}
    e.close()
    if mlp:
        # MLP hop: tensor-bound; algorithmic flops per input tuple 2*12288*H + 2*H*C
        pm = w.preds[mlps[0]]
        flops_t = 2 * K4_FEATURES * pm["hidden"] + 2 * pm["hidden"] * pm["n_classes"]
        peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        ach_tf = km_tuples * flops_t / (km_ms / 1000.0) / 1e12 if km_ms > 0 else 0.0
        mtraffic, mtraffic_note = _profile_traffic("mlp_dram_traffic.json")
        roofline = {"kernel": "hydro_mlp_kernel (K4-MLP: crop gather + two chained tcgen05 GEMMs, CTA pairs)",
                    "bound": "tensor", "achieved": ach_tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach_tf / peak_tf,
                    "frac_vs_burst_peak": ach_tf / peaks["bf16_tflops"],
                    "traffic": mtraffic, "traffic_source": mtraffic_note,
                    "algorithmic_flops_per_launch": km_tuples * flops_t / max(km_n, 1),
                    "avg_launch_ms": km_ms / max(km_n, 1), "launches": km_n,
                    "share_of_step": km_ms / ms, "time_source": "device launch timers inside the timed run",
                    "mlp_ms_per_step": km_ms / args.steps, "linear_k4_ms_per_step": k4_ms / args.steps,
                    "k1_ms_per_step": k1_ms / args.steps, "k2_ms_per_step": k2c_ms / args.steps,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside the step; fp16 "
                                   "operands of layer 1 run at the bf16 rate)"}
    else:
        k4_name = ("hydro_classifier_kernel (K4: cp.async-staged crop gather, A in shared memory, tcgen05 linear head)"
                   if os.environ.get("HYDRO_K4_LEGACY") == "1" else
                   "hydro_classifier_tm_kernel (K4-T: bulk-copy-staged crop gather, A in tensor memory, tcgen05 "
                   "linear head)")
        roofline = {"kernel": k4_name,
                    "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_note,
                    "algorithmic_bytes_per_launch": k4_bytes / max(k4_n, 1),
                    "algorithmic_bytes_per_tuple": K4_BYTES_PER_TUPLE, "classifier_tuples_per_step": k4_tuples / args.steps,
                    "head_evaluations_per_step": k4_evals / args.steps,
                    "fused_pair": [w.preds[k]["name"] for k in pair_ks],
                    "avg_launch_ms": k4_ms / max(k4_n, 1), "launches": k4_n,
                    "share_of_step": k4_ms / ms, "time_source": "device launch timers inside the timed run",
                    "k2_ms_per_step": k2c_ms / args.steps,
                    "k1_ms_per_step": k1_ms / args.steps, "k4_ms_per_step": k4_ms / args.steps,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "_fallback" not in peaks else "fallback"}
        if traffic and k4_n and k4_ms > 0:
            # the bytes K4 actually moves (ncu dram__bytes per launch, profiles/k4_dram_traffic.json)
            # over this run's live launch time: nearest sampling touches whole DRAM bursts around
            # the 64 sampled pixels of a row, so this exceeds the algorithmic rate above
            tgbs = traffic / (k4_ms / k4_n / 1000.0) / 1e9
            roofline.update({"traffic_gbs": tgbs, "traffic_frac": tgbs / peaks["hbm_gbs"]})
        if hsv:  # the HSV colour hop (K4-HSV) is ALU work: its own time and rate next to the linear hop
            roofline.update({"hsv_ms_per_step": kh_ms / args.steps, "hsv_launches": kh_n,
                             "hsv_kernel_tuples_per_s": kh_tuples / (kh_ms / 1000.0) if kh_ms > 0 else None})
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "fp16" if all(op_fp16) else "bf16", "data": "synthetic",
               "config": {"workload": WORKLOAD_MLP if mlp else (WORKLOAD_HSV if hsv else WORKLOAD),
                          "weights": args.weights + ((" (every weight fp16-exact: fp16 operands, the same products)"
                                                      if not any(op_scale) else
                                                      f" (general bf16 heads tiled as 2^k W, k = {op_scale}: fp16-exact, "
                                                      "logits scaled back by 2^-k exactly; fp16 operands, the same "
                                                      "products)") if all(op_fp16) else " (bf16 operands)"),
                          "tuples_per_step": world * TUPLES_PER_STEP,
                          "batch_tuples": TUPLES_PER_STEP, "policy": "score (cost/(1-sel)), measured costs",
                          "l2": "inputs larger than L2: 2.83 GB frame pool + 6 rotating 22 MB tuple batches",
                          "parallelism": f"dp{world}", "final_order": [w.preds[k]["name"] for k in order],
                          "selectivity": sel, "cost_sm_cycles_per_tuple": cost},
               "roofline": roofline,
               "cpu_baseline": cpu,
               "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": int(sum(d2h) / max(len(d2h), 1))},
               "clocks": clk.summary(), "gpu_launches": launches, "paper_context": PAPER_CONTEXT}
        print(json.dumps(out))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_orders(args):
    """--workload orders: the eddy against every fixed order (the
    adaptive routing claim).  cfg2's query over 1M tuples per step: each of the 3! fixed predicate
    orders (policy fixed, no routing decisions) and the adaptive score policy (measured costs and
    selectivities), device-timed the same way as the headline run; reports each order's tuples/s, the
    order the eddy settles on and its throughput relative to the best fixed order."""
    import itertools

    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from synth import workload

    torch.cuda.set_device(0)
    B.build()
    w = workload("cfg2", weights=args.weights)
    frames = w.frames(device="cuda")
    stream = torch.cuda.current_stream()
    batches = [w.tuples(id_start=b * TUPLES_PER_STEP, n=TUPLES_PER_STEP, device="cuda") for b in range(ROTATING_BATCHES)]
    res_ids = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
    res_bb = torch.empty((1 << 20, 4), dtype=torch.int16, device="cuda")
    names = [p["name"] for p in w.preds]

    def measure(order):
        e = H.Eddy(frames=frames, policy="fixed" if order else "score", warmup_tuples=65536,
                   max_batch_tuples=1 << 20, max_inflight=4, stream=stream)
        for p in w.preds:
            e.add_predicate(p)
        if order:
            e.set_fixed_order(list(order))

        def run(k, off):
            pend = []
            for st in range(k):
                pend.append(e.submit(batches[(off + st) % ROTATING_BATCHES]))
                if len(pend) >= 3:
                    e.collect_into(pend.pop(0), res_ids, res_bb)
            for bid in pend:
                e.collect_into(bid, res_ids, res_bb)

        run(max(args.warmup, 3), 0)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        run(args.steps, 1)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / args.steps
        final = [names[k] for k in e.order()]
        e.close()
        return TUPLES_PER_STEP / (ms / 1000.0), ms, final

    fixed = {}
    for order in itertools.permutations(range(len(w.preds))):
        tps, ms, _ = measure(order)
        fixed[" -> ".join(names[k] for k in order)] = {"tuples_per_s": tps, "ms_per_step": ms}
    tps, ms, final = measure(None)
    best = max(fixed.items(), key=lambda kv: kv[1]["tuples_per_s"])
    worst = min(fixed.items(), key=lambda kv: kv[1]["tuples_per_s"])
    out = {"metric": "tuples/s of the adaptive eddy (score policy) against every fixed predicate order, cfg2",
           "value": tps, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16", "data": "synthetic",
           "config": {"workload": WORKLOAD, "weights": args.weights},
           "eddy_final_order": final, "fixed_orders": fixed,
           "best_fixed": best[0], "eddy_over_best_fixed": tps / best[1]["tuples_per_s"],
           "best_over_worst_fixed": best[1]["tuples_per_s"] / worst[1]["tuples_per_s"]}
    print(json.dumps(out))


def run_route(args):
    """--workload rroute: evidence run for the route/compaction kernel K1 (SURVEY.md §8(d) R-route):
    label='dog' (0.5) AND HASH (0.5, 1 unit) AND HASH (0.5, 1 unit) over 16M-tuple batches (352 MB of
    columns per batch, far above L2), 96M tuples per step.  All three predicates are cheap, so one K1
    launch per batch runs the whole chain and emits (id, bbox).  Algorithmic bytes per input tuple:
    label 2 B + id 8 B (the fused run loads ids once for every alive position) + 16 B per emitted row."""
    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from synth import hash_pred, label_pred, workload

    torch.cuda.set_device(0)
    B.build()
    batch, nb = 1 << 24, 6
    w = workload("cfg2", n=batch)
    w.preds = [label_pred(), hash_pred(31, 0.5, units=1), hash_pred(32, 0.5, units=1)]
    stream = torch.cuda.current_stream()
    e = H.Eddy(policy="score", warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4, stream=stream)
    for p in w.preds:
        e.add_predicate(p)
    batches = [w.tuples(id_start=b * batch, n=batch, device="cuda") for b in range(nb)]
    res_ids = torch.empty(batch, dtype=torch.int64, device="cuda")
    res_bb = torch.empty((batch, 4), dtype=torch.int16, device="cuda")
    outs = []

    def run_steps(k):
        pend = []
        for s in range(k * nb):
            pend.append(e.submit(batches[s % nb]))
            if len(pend) >= 3:
                outs.append(e.collect_into(pend.pop(0), res_ids, res_bb))
        for bid in pend:
            outs.append(e.collect_into(bid, res_ids, res_bb))

    run_steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outs.clear()
    with ClockSampler(0) as clk:
        ev0.record(stream)
        run_steps(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    n_out = sum(outs)
    e.set_kernel_timing(True)
    outs.clear()
    run_steps(args.steps)
    k1_ms, k1_n = e.kernel_time(0)
    k2_ms, k2_n = e.kernel_time(3)
    e.set_kernel_timing(False)
    tuples = args.steps * nb * batch
    # SURVEY.md §8(d) R-route: 2 (label) + 4 (id of the 1/2 label-passing tuples) + 2 (id of the 1/4
    # passing the first HASH) = 8 algorithmic bytes per input tuple
    alg_bytes = tuples * 8
    peaks = _peaks()
    achieved = alg_bytes / ((k1_ms + k2_ms) / 1000.0) / 1e9
    achieved_step = alg_bytes / (ms / 1000.0) / 1e9
    # bytes K1 + K2 actually move per 16M-tuple batch (ncu dram__bytes of one working launch of each,
    # profiles/route_k{1,2}_dram_traffic.json stamped with the sources they were captured on)
    t1, n1_note = _profile_traffic("route_k1_dram_traffic.json")
    t2, n2_note = _profile_traffic("route_k2_dram_traffic.json")
    route_traffic = (t1 + t2) if (t1 and t2) else None
    route_traffic_note = n1_note + "; " + n2_note
    route_traffic_frac = (route_traffic * args.steps * nb / ((k1_ms + k2_ms) / 1000.0) / 1e9 / peaks["hbm_gbs"]
                          if route_traffic and k1_ms + k2_ms > 0 else None)
    out = {"metric": "tuples/s through the 3-predicate cheap conjunction (R-route evidence for K1+K2)",
           "value": tuples / (ms / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u64", "data": "synthetic",
           "config": {"workload": "R-route: label=dog AND hash(0.5) AND hash(0.5), 16M-tuple batches x 6 per step",
                      "l2": "inputs larger than L2 (352 MB of columns per batch)", "results_per_step": n_out // max(args.steps, 1)},
           "roofline": {"kernel": ("hydro_route_kernel + hydro_compact_kernel (K1 evaluate + K2 compact/emit)"
                                   if k2_n else "hydro_route_emit_kernel (K1F: evaluate + emit in one pass, "
                                   "decoupled look-back)"),
                        "bound": "hbm", "achieved": achieved,
                        "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                        "achieved_over_step": achieved_step, "frac_over_step": achieved_step / peaks["hbm_gbs"],
                        "traffic": route_traffic, "traffic_source": route_traffic_note,
                        "traffic_bytes_per_tuple": route_traffic / batch if route_traffic else None,
                        "traffic_frac": route_traffic_frac, "algorithmic_bytes_per_tuple": 8,
                        "bytes_note": "SURVEY.md §8(d): 2 B label + 8 B id x 1/2 + 8 B id x 1/4; the emitted "
                                      "(id, bbox) rows (16 B x 1/8 read + written) are not counted",
                        "k1_ms_per_step": k1_ms / args.steps, "k2_ms_per_step": k2_ms / args.steps,
                        "k1_launches": k1_n, "k2_launches": k2_n},
           "clocks": clk.summary()}
    e.close()
    # routing + compaction alone (no UDF arithmetic): label='dog' then emit; K1 reads the label
    # column (2 B/tuple), K2 reads the survivors' id + bbox and writes the (id, bbox) rows
    if os.environ.get("HYDRO_ROUTE_ONLY") == "1":  # (ncu launch lists of the R-route run alone)
        print(json.dumps(out))
        return
    e = H.Eddy(policy="score", warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4, stream=stream)
    e.add_predicate(label_pred())
    run_steps(2)
    torch.cuda.synchronize()
    e.set_kernel_timing(True)
    outs.clear()
    run_steps(args.steps)
    l1_ms, l1_n = e.kernel_time(0)
    l2_ms, l2_n = e.kernel_time(3)
    e.set_kernel_timing(False)
    e.close()
    lbytes = tuples * 2 + 32 * sum(outs)
    lach = lbytes / ((l1_ms + l2_ms) / 1000.0) / 1e9
    out["roofline_label_only"] = {
        "kernel": ("hydro_route_kernel + hydro_compact_kernel" if l2_n else "hydro_route_emit_kernel (K1F)")
                  + " on label='dog' alone (routing + compaction, no UDF arithmetic)",
        "bound": "hbm", "achieved": lach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
        "frac": lach / peaks["hbm_gbs"], "algorithmic_bytes_per_tuple": lbytes / tuples,
        "k1_ms_per_step": l1_ms / args.steps, "k2_ms_per_step": l2_ms / args.steps,
        "launches": l1_n + l2_n}
    print(json.dumps(out))


def run_uc2(args):
    """--workload uc2: reuse-aware routing evidence.  UC2
    scaled by 1000: 15M tuples in 1M-tuple routing batches, two expensive HASH stand-ins for the
    ObjectDetector / HardHatDetector (1024 fmix32 rounds each, selectivity 0.5) whose verdicts were
    cached by exploratory queries over ids (1M, 7M) and (8M, 14M) (hydro_cache_fill, untimed).  The
    same query runs under three policies -- the baseline's fixed order, cost-driven (measured costs)
    and reuse-aware cost-driven -- each timed over the 15 batches after a warm-up pass."""
    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from synth import workload

    torch.cuda.set_device(0)
    B.build()
    frames = None
    if args.workload == "uc2cls":
        # the cached detectors are CLASSIFIER hops (K0c split + K4-T on the uncached tuples): the
        # dog query's breed (C=120) and colour (C=10) linear heads on 64x64 nearest crops
        n, batch, scale = 3_000_000, 1_000_000, 200
        wd = workload("cfg2", n=n)
        w = wd
        w.preds = [wd.preds[1], wd.preds[2]]
        frames = wd.frames(device="cuda")
        detectors = "breed (C=120) + colour (C=10) linear heads on 64x64 nearest crops"
    else:
        n, batch, scale, units = 15_000_000, 1_000_000, 1000, 1024
        w = workload("uc2", n=n)
        for p in w.preds:  # expensive detectors: the UDF cost, not the routing overhead, must dominate
            p["units"], p["declared_cost"] = units, float(units)
        detectors = "2 HASH detectors (1024 rounds, sel 0.5)"
    t = w.tuples(device="cuda")
    ranges = [(1000 * scale, 7000 * scale), (8000 * scale, 14000 * scale)]
    stream = torch.cuda.current_stream()
    res_ids = torch.empty(batch, dtype=torch.int64, device="cuda")
    res_bb = torch.empty((batch, 4), dtype=torch.int16, device="cuda")
    times, results = {}, {}
    for policy in ("fixed", "cost", "reuse"):
        e = H.Eddy(frames=frames, policy=policy, warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4,
                   stream=stream)
        for p in w.preds:
            e.add_predicate(p)
        for k, (lo, hi) in enumerate(ranges):
            e.cache_enable(k, n)
            for a in range(lo + 1, hi, batch):
                e.cache_fill(k, t.slice(a, min(a + batch, hi)))
        if policy == "fixed":
            e.set_fixed_order([0, 1])

        def one_pass():
            pend, total = [], 0
            for a in range(0, n, batch):
                pend.append(e.submit(t.slice(a, a + batch)))
                if len(pend) >= 3:
                    total += e.collect_into(pend.pop(0), res_ids, res_bb)
            for bid in pend:
                total += e.collect_into(bid, res_ids, res_bb)
            return total

        for _ in range(max(args.warmup, 1)):
            one_pass()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms, tot = [], 0
        for _ in range(args.steps):
            ev0.record(stream)
            tot = one_pass()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        times[policy] = sorted(ms)[len(ms) // 2]
        results[policy] = tot
        e.close()
    assert len(set(results.values())) == 1, results  # the policy never changes the result
    out = {"metric": "tuples/s through the UC2 query under reuse-aware routing (SURVEY.md §8(f) f2 evidence)",
           "value": n / (times["reuse"] / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": times["reuse"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u64", "data": "synthetic",
           "config": {"workload": f"uc2 x{scale}: {n // 1_000_000}M tuples, 1M-tuple batches, {detectors}, "
                                  f"verdicts cached for ids ({ranges[0][0]}, {ranges[0][1]}) / ({ranges[1][0]}, "
                                  f"{ranges[1][1]}) by hydro_cache_fill (untimed)",
                      "results": results["reuse"]},
           "policies_ms": times,
           "speedup_reuse_vs_fixed": times["fixed"] / times["reuse"],
           "speedup_reuse_vs_cost": times["cost"] / times["reuse"],
           "paper_uc2_context": "PAPER.md:626-628: reuse-aware 386.81 s vs baseline 482.41 s (1.25x), "
                                "cost-driven only 545.03 s (reuse-aware 1.41x faster); other hardware, real detectors"}
    print(json.dumps(out))


def run_area(args):
    """--workload area: data-aware tile scheduling evidence (
    DESIGN.md R28).  cfg4's query (label, area-weighted HASH, colour nearest, breed AREA) over 10M
    tuples per step in routing batches of 1M and of 256K tuples; the AREA hop (cost proportional to
    the bbox area) runs with round-robin tiles and with data-aware ranges of equal
    estimated cost (input size w*h).  Reports each mode's step time, K4 time (both
    linear heads; only the AREA hop differs), K6 time, and checks that the results are identical."""
    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from synth import workload

    torch.cuda.set_device(0)
    B.build()
    n = 10_000_000
    w = workload("cfg4", n=n)
    frames = w.frames(device="cuda")
    t = w.tuples(device="cuda")
    stream = torch.cuda.current_stream()
    out_modes = {}
    for batch in (1 << 20, 1 << 18):
        res_ids = torch.empty(batch, dtype=torch.int64, device="cuda")
        res_bb = torch.empty((batch, 4), dtype=torch.int16, device="cuda")
        for balance in ("round_robin", "data_aware"):
            e = H.Eddy(frames=frames, policy="score", warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4,
                       stream=stream, balance=balance)
            for p in w.preds:
                e.add_predicate(p)

            def one_pass():
                pend, total = [], 0
                for a in range(0, n, batch):
                    pend.append(e.submit(t.slice(a, min(a + batch, n))))
                    if len(pend) >= 3:
                        total += e.collect_into(pend.pop(0), res_ids, res_bb)
                for bid in pend:
                    total += e.collect_into(bid, res_ids, res_bb)
                return total

            for _ in range(max(args.warmup, 1)):
                one_pass()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ms, tot = [], 0
            for _ in range(args.steps):
                ev0.record(stream)
                tot = one_pass()
                ev1.record(stream)
                torch.cuda.synchronize()
                ms.append(ev0.elapsed_time(ev1))
            e.set_kernel_timing(True)
            one_pass()
            k4_ms, _ = e.kernel_time(1)
            k6_ms, k6_n = e.kernel_time(6)
            e.set_kernel_timing(False)
            order = [w.preds[k]["name"] for k in e.order()]
            e.close()
            out_modes[f"{balance}@{batch}"] = {"ms_per_step": sorted(ms)[len(ms) // 2], "k4_ms_per_step": k4_ms,
                                               "k6_ms_per_step": k6_ms, "k6_launches": k6_n, "results": tot,
                                               "final_order": order}
    for batch in (1 << 20, 1 << 18):
        a, b = out_modes[f"round_robin@{batch}"], out_modes[f"data_aware@{batch}"]
        assert a["results"] == b["results"], (a, b)  # the schedule never changes the result
    best = out_modes[f"data_aware@{1 << 20}"]
    # the AREA hop alone (cfg4's AREA breed head on the first 1M tuples, every tuple a crop; K4's
    # 20-converter-warp AREA instance): device launch timers; algorithmic bytes = the crop's source
    # pixels (3 w h) + 16 B of metadata per crop
    na = 1 << 20
    ta = t.slice(0, na)
    ea = H.Eddy(frames=frames, policy="fixed", warmup_tuples=0, max_batch_tuples=na, stream=stream)
    ea.add_predicate(w.preds[3])
    res_ids = torch.empty(na, dtype=torch.int64, device="cuda")
    res_bb = torch.empty((na, 4), dtype=torch.int16, device="cuda")
    for _ in range(2):
        ea.collect_into(ea.submit(ta), res_ids, res_bb)
    torch.cuda.synchronize()
    ea.device_time(1, reset=True)
    ea.device_items(1, reset=True)
    for _ in range(max(args.steps, 3)):
        ea.collect_into(ea.submit(ta), res_ids, res_bb)
    torch.cuda.synchronize()
    a_ms, a_n = ea.device_time(1)
    a_crops = ea.device_items(1)
    ea.close()
    bb = ta.bbox.long()
    a_bytes_per_crop = float((3 * (bb[:, 2] - bb[:, 0]) * (bb[:, 3] - bb[:, 1])).double().mean().item()) + 16.0
    a_gbs = a_crops * a_bytes_per_crop / (a_ms / 1000.0) / 1e9 if a_ms > 0 else 0.0
    peaks = _peaks()
    roofline = {"kernel": "hydro_classifier_kernel<.., AREA, 20 converter warps> (row-cooperative AREA converter, "
                          "tcgen05 linear head), the AREA hop alone on 1M cfg4 crops",
                "bound": "hbm", "achieved": a_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": a_gbs / peaks["hbm_gbs"], "crops_per_s": a_crops / (a_ms / 1000.0) if a_ms > 0 else None,
                "algorithmic_bytes_per_crop": a_bytes_per_crop, "launches": a_n,
                "time_source": "device launch timers",
                "note": "instruction-issue bound in practice (ncu: issue active 76%, DRAM 15% of peak; "
                        "profiles/round2_ncu_summary.md)"}
    out = {"metric": "tuples/s through cfg4 with data-aware tile scheduling of the AREA hop (SURVEY.md §8(f) f4)",
           "value": n / (best["ms_per_step"] / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": best["ms_per_step"], "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
           "config": {"workload": "cfg4: 10M tuples per step (label, area-weighted HASH, colour nearest, breed "
                                  "AREA), routing batches of 1M and 256K", "frames": "1024 x 720x1280x3"},
           "modes": out_modes, "roofline": roofline,
           "speedup_data_aware_1M": out_modes[f"round_robin@{1 << 20}"]["ms_per_step"] / best["ms_per_step"],
           "speedup_data_aware_256K": out_modes[f"round_robin@{1 << 18}"]["ms_per_step"]
           / out_modes[f"data_aware@{1 << 18}"]["ms_per_step"],
           "paper_uc4_context": "PAPER.md:914-916: data-aware 1238.98 s vs round-robin 1652.67 s (1.33x) for LLM "
                                "workers on a 32-core CPU; other hardware and workload"}
    print(json.dumps(out))


def _flow_shop(rows):
    """Makespan of batches through serial workers in a fixed order (the model the bench compares
    the measured times with): C[b][i] = max(C[b][i-1], C[b-1][i]) + t[b][i]."""
    prev = None
    for row in rows:
        cur = []
        for i, t in enumerate(row):
            cur.append(max(cur[i - 1] if i else 0.0, prev[i] if prev else 0.0) + t)
        prev = cur
    return prev[-1] if prev else 0.0


def run_concurrent(args):
    """--workload concurrent: cost-driven routing over concurrent workers (
    PAPER.md:320-365; R29).  Two scenarios, each predicate a worker on its own half of the
    SMs (own context, stream and green-context SM partition); batches flow through the workers in
    the policy's order, consecutive batches overlapping:
      example: the paper's example (colour: cost 1, selectivity 0.6; breed: cost 2, selectivity
               0.1) as HASH stand-ins with 512 / 1024 rounds, 16M tuples in 1M
               batches (the headline line);
      dog:     the UC1 classifiers themselves -- DogColorClassifier as the HSV heuristic and the
               breed linear head (C=120) on 64x64 crops of a coloured-block frame pool, 2M dog
               detections in 256K batches.
    Timed per scenario: cost-, score- and selectivity-driven routing, and the sequential eddy on all
    SMs (one context, score policy) for reference; plus the flow-shop model's prediction from the
    warmup's measured costs and selectivities."""
    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from paper_2403_14902_b200.pipeline import ConcurrentEddy
    from synth import hash_pred, workload

    torch.cuda.set_device(0)
    B.build()
    main = torch.cuda.current_stream()

    def timed(fn):
        fn()  # warm-up pass
        torch.cuda.synchronize()
        ms = []
        for _ in range(args.steps):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(main)
            out = fn()  # returns after the last batch's results were collected (all work done)
            ev1.record(main)
            torch.cuda.synchronize()
            ms.append(ev0.elapsed_time(ev1))
        return sorted(ms)[len(ms) // 2], out

    def scenario(preds, t, n, batch, frames=None, policies=("cost", "score", "selectivity")):
        batches = [t.slice(a, min(a + batch, n)) for a in range(0, n, batch)]
        res_ids = torch.empty(batch, dtype=torch.int64, device="cuda")
        res_bb = torch.empty((batch, 4), dtype=torch.int16, device="cuda")
        modes = {}
        for policy in policies:
            pol, part = (policy.split("@") + ["green"])[:2]
            ce = ConcurrentEddy(preds, frames=frames, policy=pol, max_batch_tuples=batch, partition=part)
            order = ce.warmup(batches[0])
            c, sel = list(ce.cost_per_tuple), list(ce.selectivity)
            ms, out = timed(lambda: sum(r[0] for r in ce.run(batches, res_ids, res_bb)))
            rows = []  # flow-shop model: stage i sees the fraction the earlier stages passed
            for b in batches:
                alive, row = float(len(b)), []
                for k in order:
                    row.append(alive * c[k])
                    alive *= sel[k]
                rows.append(row)
            modes[policy] = {"ms_per_pass": ms, "order": [preds[k]["name"] for k in order], "results": out,
                             "cycles_per_tuple_per_worker": [round(x, 2) for x in c],
                             "selectivity": [round(x, 4) for x in sel], "model_cycles": _flow_shop(rows),
                             "sms": ce.sms, "partition": part}
            ce.close()
        seq = H.Eddy(frames=frames, policy="score", warmup_tuples=65536, max_batch_tuples=batch, max_inflight=4,
                     stream=main)
        for p in preds:
            seq.add_predicate(p)

        def seq_pass():
            pend, tot = [], 0
            for b in batches:
                pend.append(seq.submit(b))
                if len(pend) >= 3:
                    tot += seq.collect_into(pend.pop(0), res_ids, res_bb)
            for bid in pend:
                tot += seq.collect_into(bid, res_ids, res_bb)
            return tot

        ms_seq, tot_seq = timed(seq_pass)
        modes["sequential_all_sms_score"] = {"ms_per_pass": ms_seq, "order": [preds[k]["name"] for k in seq.order()],
                                             "results": tot_seq}
        seq.close()
        assert len({m["results"] for m in modes.values()}) == 1, modes  # routing never changes the result
        return modes

    n, batch, units = 16_000_000, 1 << 20, 512
    ex_preds = [hash_pred(31, 0.6, units=units, name="colour (cost 1, sel 0.6)"),
                hash_pred(32, 0.1, units=2 * units, name="breed (cost 2, sel 0.1)")]
    ex = scenario(ex_preds, workload("cfg1", n=n).tuples(device="cuda"), n, batch,
                  policies=("cost", "score", "selectivity", "cost@grid", "score@grid"))
    wd = workload("hsv")
    frames = wd.frames(device="cuda")
    nd, bd = 2_000_000, 1 << 18
    td = wd.tuples(n=nd, device="cuda")
    dog_preds = [wd.preds[2], wd.preds[1]]  # colour (HSV heuristic), breed (linear C=120)
    dog = scenario(dog_preds, td, nd, bd, frames=frames)
    cost, score = ex["cost"], ex["score"]
    out = {"metric": "tuples/s through the paper's two-predicate example on concurrent workers (SURVEY.md §8(f) f3)",
           "value": n / (cost["ms_per_pass"] / 1000.0), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": 1, "ms_per_step": cost["ms_per_pass"], "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": {"workload": "concurrent: colour HASH (512 rounds, sel 0.6) and breed HASH (1024 rounds, sel "
                                  "0.1), one worker per predicate on its own half of the SMs (green-context "
                                  "partitions; @grid = grid caps only), 16M tuples in 1M batches"},
           "modes": ex,
           "speedup_cost_vs_score": score["ms_per_pass"] / cost["ms_per_pass"],
           "model_speedup_cost_vs_score": score["model_cycles"] / cost["model_cycles"],
           "dog_query_workers": {"workload": "DogColorClassifier (HSV heuristic) and DogBreedClassifier (linear "
                                             "C=120) as two workers, 2M detections in 256K batches, coloured-block frames",
                                 "modes": dog,
                                 "tuples_per_s": {k: nd / (v["ms_per_pass"] / 1000.0) for k, v in dog.items()}},
           "paper_context": "PAPER.md:357-359: 20 (score/selectivity-driven) vs 14 (cost-driven) time units for 10 items"}
    print(json.dumps(out))


def run_small(args):
    """--workload small: the latency- and adaptation-bound configs.
    cfg1: 10k tuples, two HASH predicates (sel 0.5 / 0.1, 1 / 10 units), STATIC statistics, one batch:
          microseconds per batch (submit -> rows on the host), median over repetitions.
    cfg3: 1M tuples in 64K batches, three HASH predicates (2 / 4 / 8 units) whose selectivities swap
          at id 500,000 (0.9, 0.5, 0.1 -> 0.1, 0.5, 0.9): tuples/s, the batches the score policy takes
          to reach the post-drift optimal order, and the realized cost (units x tuples evaluated,
          from the per-batch counters) against each half's optimum E(pi*) = sum_i c_i prod_{j<i} s_j."""
    import itertools

    import torch

    from paper_2403_14902_b200 import build as B
    from paper_2403_14902_b200 import hydro as H
    from synth import workload

    torch.cuda.set_device(0)
    B.build()
    stream = torch.cuda.current_stream()
    # ---- cfg1 latency
    w1 = workload("cfg1")
    t1 = w1.tuples(device="cuda")
    e = H.Eddy(policy="static", warmup_tuples=0, max_batch_tuples=len(t1), stream=stream)
    for p in w1.preds:
        e.add_predicate(p)
    # rows land in preallocated pinned host buffers (collect_into: one D2H copy, no allocation)
    out_ids = torch.empty(len(t1), dtype=torch.int64).pin_memory()
    out_bb = torch.empty((len(t1), 4), dtype=torch.int16).pin_memory()
    for _ in range(20):
        e.collect_into(e.submit(t1), out_ids, out_bb)
    lat, dev, lat_alloc = [], [], []
    for _ in range(200):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        ev0.record(stream)
        b = e.submit(t1)
        ev1.record(stream)
        n1 = e.collect_into(b, out_ids, out_bb)
        lat.append((time.perf_counter() - h0) * 1e6)
        dev.append(ev0.elapsed_time(ev1) * 1e3)
    for _ in range(100):  # the allocating collect (new pageable result tensors per batch), for reference
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        ids, _ = e.collect(e.submit(t1))
        lat_alloc.append((time.perf_counter() - h0) * 1e6)
    assert len(ids) == n1
    launches = e.launch_count()
    e.close()
    # ---- cfg3 adaptation
    w3 = workload("cfg3")
    n3, b3 = w3.n, w3.batch_tuples
    t3 = w3.tuples(device="cuda")
    units = [p["units"] for p in w3.preds]
    sel_before, sel_after = [0.9, 0.5, 0.1], [0.1, 0.5, 0.9]

    def e_cost(order, sel):
        tot, alive = 0.0, 1.0
        for k in order:
            tot += units[k] * alive
            alive *= sel[k]
        return tot

    best_before = min(itertools.permutations(range(3)), key=lambda o: e_cost(o, sel_before))
    best_after = min(itertools.permutations(range(3)), key=lambda o: e_cost(o, sel_after))
    res = {}
    for policy in ("score", "static"):
        e = H.Eddy(policy=policy, warmup_tuples=w3.warmup_tuples, max_batch_tuples=b3, stream=stream)
        for p in w3.preds:
            e.add_predicate(p)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        infos, total = [], 0
        res_ids = torch.empty(b3, dtype=torch.int64, device="cuda")
        res_bb = torch.empty((b3, 4), dtype=torch.int16, device="cuda")
        pend = []

        def retire(bid):
            infos.append(e.batch_info(bid))  # (before collect: the report lives in the batch's slot)
            return e.collect_into(bid, res_ids, res_bb)  # rows stay on the device

        for a in range(0, n3, b3):
            if a == b3:  # batch 0 (first submit: buffer allocation, warmup slice) is not timed
                total += retire(pend.pop(0))
                torch.cuda.synchronize()
                ev0.record(stream)
            pend.append(e.submit(t3.slice(a, min(a + b3, n3))))
            if len(pend) >= 3:  # three batches in flight (the order of each is still decided on the device in turn)
                total += retire(pend.pop(0))
        while pend:
            total += retire(pend.pop(0))
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        e.close()
        drift_batch = (n3 // 2) // b3
        lag = next((i - drift_batch for i in range(drift_batch, len(infos))
                    if tuple(infos[i]["order_used"]) == tuple(best_after)), None)
        realized = sum(sum(u * x for u, x in zip(units, inf["tuples_in"])) for inf in infos)
        optimal = sum(e_cost(best_before if (i * b3) < n3 // 2 else best_after, sel_before if (i * b3) < n3 // 2 else sel_after)
                      * min(b3, n3 - i * b3) for i in range(len(infos)))
        res[policy] = {"tuples_per_s": (n3 - b3) / (ms / 1000.0), "ms": ms, "timed": "batches 1..15", "results": total,
                       "orders": [inf["order_used"] for inf in infos], "adaptation_lag_batches": lag,
                       "realized_cost_units": realized, "optimal_cost_units": optimal,
                       "regret": realized / optimal}
    out = {"metric": "latency (cfg1) and adaptation (cfg3) of the eddy (SURVEY.md §8(d))",
           "value": statistics.median(lat), "unit": "us/batch", "n_gpus": 1, "steps": 200, "warmup": 20,
           "ms_per_step": statistics.median(lat) / 1000.0, "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "u64", "data": "synthetic",
           "config": {"workload": "cfg1: 10k tuples, HASH 0.5/0.1 (1/10 units), STATIC, one batch; cfg3: 1M tuples, "
                                  "64K batches, selectivity drift at id 500k"},
           "cfg1": {"us_per_batch_host": statistics.median(lat), "us_per_batch_device": statistics.median(dev),
                    "host_path": "submit (device columns) -> collect_into preallocated pinned host buffers",
                    "us_per_batch_host_allocating_collect": statistics.median(lat_alloc),
                    "results": n1, "launches_total": launches},
           "cfg3": {"best_order_before": list(best_before), "best_order_after": list(best_after), **res}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--e2e-depth", type=int, default=2, help="batches in flight in the e2e (host buffer) run")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hydro", choices=["hydro", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--weights", default="grid", choices=["grid", "bf16"],
                    help="classifier heads: fp16-exact 'grid' weights or general bf16 weights (N(0, 2.5e-4^2))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "rroute", "mlp", "uc2", "uc2cls", "hsv", "area", "concurrent",
                                                          "small", "orders"],
                    help="cfg2 = the BASELINE metric (default); rroute = K1 HBM evidence run; "
                         "mlp = cfg2 with the 12288-512-120 MLP breed head (SURVEY.md §8(f) f1, tensor roofline)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "rroute":
        run_route(args)
    elif args.workload in ("uc2", "uc2cls"):
        run_uc2(args)
    elif args.workload == "area":
        run_area(args)
    elif args.workload == "concurrent":
        run_concurrent(args)
    elif args.workload == "small":
        run_small(args)
    elif args.workload == "orders":
        run_orders(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
