"""Benchmark of the indirect-convolution hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl icv|reference] [--config cfg2]

One "step" = one pass of the hot path (the indirect-GEMM convolution, the
indirection buffer and packed filter already built, as in the reference
harness bench.py:156-161) over one batch of the BASELINE workload.  Default
workload: BASELINE.json configs[1] (cfg2: bf16 64x28x28x128 -> 128, 3x3).

Multi-GPU (torchrun, one process per GPU, NCCL): the batch dimension is
partitioned — every rank convolves its own 64 images (weak scaling) with the
filter packed once on rank 0 and replicated by one NCCL broadcast (the only
collective; it is setup, outside the timed region).  Timing: CUDA events
around every step on the launching stream, L2 flushed (256 MiB write)
between steps, max over ranks.

``--impl reference`` times the reference's own CPU algorithm for the path
(the numpy port in oracle/, which restates convbench's indirect_conv;
the reference itself is pure Python and cannot travel to the GPU box) on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "which": "fallback"}


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        p["which"] = "measured"
    except OSError:
        p = dict(PEAKS_FALLBACK)
    try:   # int8 / fp32 peaks measured on a B200 of this pool (tools/measure_peaks.py)
        with open(os.path.join(ROOT, "profiles", "peaks_extra.json")) as f:
            extra = json.load(f)
        p["int8_tops"] = extra.get("int8_tops")
        p["fp32_tflops"] = extra.get("fp32_tflops")
    except (OSError, ValueError):
        pass
    return p


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms (NVML) while running;
    falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device_index: int):
        self.idx = device_index
        self.samples: list[tuple[float, float, int, float]] = []
        self.stop_evt = threading.Event()
        self.thread = None
        self.marks: list[tuple[str, int]] = []

    def mark(self, name: str):
        self.marks.append((name, len(self.samples)))

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)

            def run():
                while not self.stop_evt.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                        self.samples.append((float(sm), float(mx), int(rs), pw))
                    except Exception:  # pragma: no cover - driver dependent
                        pass
                    time.sleep(0.005)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def stop(self, window: tuple[str, str] | None = None) -> dict | None:
        self.stop_evt.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        rows = self.samples
        if window is not None:
            idx = dict(self.marks)
            lo, hi = idx.get(window[0], 0), idx.get(window[1], len(rows))
            if hi > lo:
                rows = rows[lo:hi]
        if not rows:
            return None
        reasons = sorted({n for r in rows for n, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": round(max(r[3] for r in rows), 1), "samples": len(rows),
                "window": "timed steps" if window else "whole run", "reasons": reasons}


# ---------------------------------------------------------- CPU reference arm
def _init_worker():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["MKL_NUM_THREADS"] = "1"


def _cpu_worker(args):
    """One image of the workload through the oracle port (restates
    convbench.indirect: _compute_offsets + indirect_conv).  Returns seconds
    spent in the convolution only (IB build outside timing, bench.py:156-161)."""
    name, img = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import conv as oconv
    from oracle import ib as oib
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    s = w.in_shape
    oh, ow = w.out_hw
    x = w.input_host(img, img + 1)
    wt = w.filter_host()
    if w.dtype == "bf16":
        x, wt = oconv.bf16_round(x), oconv.bf16_round(wt)
    offs = oib.compute_offsets((1, s.h, s.w, s.c), w.params, oh, ow, 1, 4)
    t0 = time.perf_counter()
    if w.dtype == "u8":
        from oracle import quant as oq
        q = w.quant
        oq.indirect_conv_u8(x, np.full(s.c, q.input_zero_point, np.uint8), offs, w.params, wt, w.bias_host(), 1,
                            oh, ow, q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                            q.output_zero_point, q.output_scale)
    else:
        oconv.indirect_conv_f32(x, np.zeros(s.c, np.float32), offs, w.params, wt, w.bias_host(), 1, oh, ow)
    return time.perf_counter() - t0


def cpu_reference(name: str, steps: int, warmup: int, cores: int | None = None) -> dict:
    """Time the oracle port on the host cores: each step convolves one image
    per worker process (a bounded sample of the workload), wall-clock."""
    import multiprocessing as mp

    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    cores = cores or os.cpu_count() or 1
    n_img = w.in_shape.n
    per_step = min(cores, n_img)
    flops_img = w.flops // n_img
    ctx = mp.get_context("spawn")
    times = []
    with ctx.Pool(per_step, initializer=_init_worker) as pool:
        for it in range(warmup + steps):
            imgs = [(name, (it * per_step + j) % n_img) for j in range(per_step)]
            t0 = time.perf_counter()
            pool.map(_cpu_worker, imgs, chunksize=1)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    total = sum(times)
    value = flops_img * per_step * len(times) / total / 1e12
    return {"value": value, "unit": "TFLOP/s", "cores": per_step, "kind": "port",
            "sample": f"{per_step} images of {name} per step (one per worker process, OMP_NUM_THREADS=1), "
                      f"{len(times)} steps, wall clock; IB built outside timing",
            "ms_per_step": 1e3 * total / len(times)}


# ---------------------------------------------------------------- GPU arm
def setup_problem(name: str, n_lo: int, n_hi: int, device, pf_bcast=None, mr: int = 128, per_image: bool = True):
    """Upload images [n_lo, n_hi) of workload `name`, build the IB on the
    device, pack (or receive) the filter."""
    import torch

    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    s = w.in_shape
    shape = icv.Shape4(n_hi - n_lo, s.h, s.w, s.c)
    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "u8": torch.uint8}[w.dtype]
    xh = w.input_host(n_lo, n_hi)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(device).to(dt))
    p = w.params
    tile = icv.TileConfig(mr=mr)
    qp = None
    zero_fill = 0
    if w.quant is not None:
        q = w.quant
        qp = icv.QuantParams(q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                             q.output_zero_point, q.output_scale, q.output_min, q.output_max)
        zero_fill = q.input_zero_point
    bias = w.bias_host()
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                            torch.from_numpy(w.filter_host()).to(device).to(dt))
    pf = icv.pack_filter(filt, None if bias is None else torch.from_numpy(bias), p, tile, quant=qp)
    if pf_bcast is not None:
        pf_bcast(pf)
    zero = icv.make_zero_row(p.in_channels, dtype=dt, device=device, fill=zero_fill)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, per_image=per_image)
    y = icv.NhwcTensor.empty(out_shape, dtype=dt, device=device)
    return w, x, xh, pf, ib, y, tile


def make_l2_flush(device):
    """L2 flush between timed steps: write a 256 MiB buffer (evicts every line
    of the step's inputs from the 126 MB L2), then read another 256 MiB, so
    the write's dirty lines are written back HERE rather than inside the next
    timed step.  Both outside the CUDA events."""
    import torch

    wbuf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=device)
    rbuf = torch.ones(32 * 1024 * 1024, dtype=torch.int64, device=device)

    def flush():
        wbuf.fill_(1)
        torch.sum(rbuf)

    return flush


def time_steps(fn, steps: int, warmup: int, flush=None, on_timed=None):
    """Per-step CUDA-event times (ms) of fn() on the current stream, with an
    optional L2 flush before every step (outside the events)."""
    import torch

    for _ in range(warmup):
        if flush is not None:
            flush()
        fn()
    torch.cuda.synchronize()
    if on_timed is not None:
        on_timed()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush()
        starts[i].record()
        fn()
        ends[i].record()
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def roofline_for(w, ms: float, peaks: dict, sustained: bool = False) -> dict:
    """Roofline of the conv kernel: tensor-bound configs against the measured
    bf16 GEMM peak (int8 against 2x that, nominal ratio, until measured),
    HBM-bound ones against the measured copy bandwidth."""
    ridge_tflops = peaks["bf16_tflops_sustained" if sustained else "bf16_tflops"]
    if w.dtype == "u8":
        # measured int8 GEMM peak (tools/measure_peaks.py -> profiles/peaks_extra.json), else 2x bf16 (nominal)
        ridge_tflops = peaks.get("int8_tops") or 2.0 * ridge_tflops
    ai = w.flops / w.compulsory_bytes
    hbm = peaks["hbm_gbs"]
    if ai * hbm / 1e3 >= ridge_tflops and w.dtype != "f32":
        achieved = w.flops / (ms * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": round(achieved, 2), "peak": ridge_tflops, "unit": "TFLOP/s",
                "frac": round(achieved / ridge_tflops, 4)}
    achieved = w.compulsory_bytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4)}


def load_traffic(name: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the conv
    kernel from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            entry = json.load(f).get(name)
        return None if entry is None else entry["bytes"]
    except (OSError, ValueError, KeyError):
        return None


def gpu_bench(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    from paper_1907_02129_b200.workloads import CONFIGS
    from paper_1907_02129_b200.dist import broadcast_packed_filter

    name = args.config
    w0 = CONFIGS[name]
    per_rank = w0.in_shape.n                      # weak scaling: fixed images per GPU
    big = w0.with_batch(per_rank * world)

    # host input of this rank's shard (images [rank*per_rank, (rank+1)*per_rank) of the global batch)
    def bcast(pf):
        if world > 1:
            broadcast_packed_filter(pf, src=0)

    import paper_1907_02129_b200.workloads as wl
    wl.CONFIGS["_bench"] = big
    w, x, xh, pf, ib, y, tile = setup_problem("_bench", rank * per_rank, (rank + 1) * per_rank, device, bcast,
                                              mr=args.mr, per_image=args.ib == "per-image")
    flush = make_l2_flush(device)

    def step():
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)

    peaks = load_peaks()
    sampler = ClockSampler(local).start() if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    times = time_steps(step, args.steps, args.warmup, flush,
                       on_timed=(lambda: sampler.mark("t0")) if sampler else None)
    if sampler:
        sampler.mark("t1")
    launches = _lib.launch_count() - launches0 - args.warmup
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()

    # ---- end-to-end through the public API with host buffers ----
    # The step's input goes host -> device and its output device -> host
    # every step.  The batch is cut into image chunks, each with its own
    # (per-image, batch-invariant) indirection buffer bound to its slice of
    # the persistent input buffer, so chunk i's H2D, chunk i-1's convolution
    # and chunk i-2's D2H overlap on three streams -- how a caller streaming
    # batches through indirect_conv would run it.
    dt = x.dtype
    x_pinned = torch.from_numpy(xh).to(dt).pin_memory() if dt != torch.uint8 else torch.from_numpy(xh).pin_memory()
    y_pinned = torch.empty(y.data.numel(), dtype=dt).pin_memory()
    n_img = x.shape.n
    n_chunks = max(1, min(args.e2e_chunks, n_img))
    bounds = [n_img * i // n_chunks for i in range(n_chunks + 1)]
    in_img = x.shape.h * x.shape.w * x.shape.c
    out_img = y.shape.h * y.shape.w * y.shape.c
    chunks = []
    for i in range(n_chunks):
        a_, b_ = bounds[i], bounds[i + 1]
        xs = icv.NhwcTensor(icv.Shape4(b_ - a_, x.shape.h, x.shape.w, x.shape.c), x.data[a_ * in_img:b_ * in_img])
        ys = icv.NhwcTensor(icv.Shape4(b_ - a_, y.shape.h, y.shape.w, y.shape.c), y.data[a_ * out_img:b_ * out_img])
        ibs = icv.init_indirection_buffer(xs, ib.zero_row, w.params, ys.shape, tile, per_image=True)
        chunks.append((a_, b_, xs, ys, ibs))
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(device), torch.cuda.Stream(device), torch.cuda.Stream(device)
    torch.cuda.synchronize()

    def e2e_enqueue():
        cur = torch.cuda.current_stream(device)
        start = torch.cuda.Event()
        start.record(cur)
        for st_ in (s_h2d, s_cmp, s_d2h):
            st_.wait_event(start)
        for a_, b_, xs, ys, ibs in chunks:
            with torch.cuda.stream(s_h2d):
                xs.data.copy_(x_pinned[a_ * in_img:b_ * in_img], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_h2d)
            s_cmp.wait_event(ev_in)
            with torch.cuda.stream(s_cmp):
                icv.indirect_conv(xs, pf, ibs, w.params, tile, out=ys)
                ev_out = torch.cuda.Event()
                ev_out.record(s_cmp)
            s_d2h.wait_event(ev_out)
            with torch.cuda.stream(s_d2h):
                y_pinned[a_ * out_img:b_ * out_img].copy_(ys.data, non_blocking=True)
        done = torch.cuda.Event()
        done.record(s_d2h)
        cur.wait_event(done)

    # the whole step (3 streams, 3 x chunks copies/launches) is captured once
    # as a CUDA graph: one launch per step, no per-chunk host overhead
    e2e_enqueue()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(device)
    with torch.cuda.stream(cap):
        graph.capture_begin()
        e2e_enqueue()
        graph.capture_end()
    torch.cuda.synchronize()

    def e2e_step():
        graph.replay()

    e2e_times = time_steps(e2e_step, max(3, min(args.steps, 50)), max(args.warmup, 3), flush)
    e2e_total = sum(e2e_times)
    e2e_n = len(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    clocks = sampler.stop(("t0", "t1")) if sampler else None

    # correctness gate on the benchmarked output (bench.py:124-142 protocol): sampled pixels vs the oracle
    gate = None
    if rank == 0 and not args.no_gate:
        gate = correctness_gate(w, xh, pf, ib, y)

    other = {}
    if rank == 0 and world == 1 and not args.no_other:
        for oname in ("cfg1", "cfg3a", "cfg3b", "cfg4"):
            if oname == name:
                continue
            ow_, ox, _, opf, oib_, oy, otile = setup_problem(oname, 0, CONFIGS[oname].in_shape.n, device,
                                                             mr=args.mr, per_image=args.ib == "per-image")
            ot = time_steps(lambda: icv.indirect_conv(ox, opf, oib_, ow_.params, otile, out=oy),
                            max(10, args.steps // 5), 3, flush)
            oms = statistics.median(ot)
            other[oname] = {"workload": ow_.name, "dtype": ow_.dtype, "ms_per_step": round(oms, 5),
                            "value": round(ow_.flops / (oms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                            "kernel": _lib.kernel_name(ow_.params, ow_.in_shape, ox.dtype),
                            "roofline": roofline_for(ow_, oms, peaks)}
            del ox, opf, oib_, oy
        other["cfg5"] = stack_bench(device, peaks, flush)
        # the paper's comparison: the GEMM-based variant (im2row patch matrix in
        # HBM + the same tcgen05 GEMM as a 1x1 conv over it) on the headline workload
        if not w.params.is_pointwise_unit_stride():
            pm = icv.build_patch_matrix(x, w.params)
            icv.gemm_only(pm, pf, tile)

            def gemm_step():
                icv.build_patch_matrix(x, w.params, out=pm)
                icv.gemm_only(pm, pf, tile)

            gt = time_steps(gemm_step, max(10, args.steps // 5), 3, flush)
            gms = statistics.median(gt)
            other["im2col_gemm_" + name] = {
                "workload": w.name, "dtype": w.dtype, "ms_per_step": round(gms, 5),
                "value": round(w.flops / (gms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                "kernels": ["icv_im2col", _lib.kernel_name(icv.ConvParams(1, 1, in_channels=pm.cols,
                                                                            out_channels=pf.k_out),
                                                          icv.Shape4(1, 1, pm.rows, pm.cols), x.dtype)],
                "patch_matrix_mb": round(pm.allocated_bytes / 1e6, 2),
                "indirect_speedup": None,   # filled below from the headline ms
                "note": "reference im2col.py gemm_conv: patch matrix built every step (build_patch_matrix + gemm_only)"}
            del pm

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_reference(name, steps=2, warmup=1)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    flops_total = w0.flops * world * args.steps
    value = flops_total / (total_ms * 1e-3) / 1e12
    ms_step = total_ms / args.steps
    med = statistics.median(times)
    roof = roofline_for(w0, statistics.mean(times), peaks)
    for k, v in other.items():
        if k.startswith("im2col_gemm_"):
            v["indirect_speedup"] = round(v["ms_per_step"] / med, 3)
    roof["traffic"] = load_traffic(w0.name)
    roof["peak_source"] = peaks["which"] + " (MEASURED_PEAKS.json bf16_tflops burst / hbm_gbs)"
    line = {
        "metric": "conv TFLOP/s (2*N*Ho*Wo*K*R*S*C / s)",
        "value": round(value, 3),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 6),
        "ms_per_step_median": round(med, 6),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16" if w0.dtype == "bf16" else w0.dtype,
        "data": "synthetic (seeded numpy; BASELINE configs are synthetic)",
        "config": {"workload": w0.name, "batch_per_gpu": per_rank, "global_batch": per_rank * world,
                   "H": w0.in_shape.h, "W": w0.in_shape.w, "C": w0.in_shape.c, "K": w0.params.out_channels,
                   "kernel": f"{w0.params.kernel_h}x{w0.params.kernel_w}", "parallelism": f"dp{world} (batch-sharded)",
                   "mr": args.mr, "index_dtype": "int64", "ib_layout": args.ib,
                   "l2": "flushed between steps (256 MiB device write + 256 MiB read, outside the timed events)",
                   "conv_kernel": _lib.kernel_name(w0.params, w0.in_shape, x.dtype)},
        "roofline": roof,
        "e2e": {"value": round(w0.flops * world * e2e_n / (e2e_total * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
                "h2d_bytes_per_step": int(x.data.numel() * x.data.element_size()),
                "d2h_bytes_per_step": int(y.data.numel() * y.data.element_size()),
                "ms_per_step": round(e2e_total / e2e_n, 5),
                "chunks": n_chunks, "cuda_graph": True,
                "path": "pinned host input -> device (bound buffer slices), indirect_conv per image chunk, output -> "
                        "pinned host; H2D / conv / D2H of successive chunks overlap on three streams"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "gate": gate,
        "other_configs": other or None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stack_bench(device, peaks: dict, flush, batch: int = 256, passes: int = 5) -> dict:
    """cfg5: the 53-layer ResNet-50 conv stack, N=256, chained through the
    public API (paper_1907_02129_b200/stack.py); median of `passes` passes
    after 2 warm-up passes, L2 flushed before each (the activations are far
    larger than L2 anyway).  Per-layer parity is tests/test_gpu_stack.py."""
    import torch

    from paper_1907_02129_b200.stack import ResNet50Stack

    stack = ResNet50Stack(batch=batch, device=device)
    for _ in range(2):
        stack.run()
    totals, pools, per = [], [], []
    for _ in range(passes):
        flush()
        t, pool, layers = stack.timed_run()
        totals.append(t)
        pools.append(pool)
        per.append(layers)
    total = statistics.median(totals)
    conv = sum(statistics.median(p[i] for p in per) for i in range(len(stack.layers)))
    bf16, hbm = peaks["bf16_tflops"], peaks["hbm_gbs"]
    roof_ms = sum(max(l.flops / (bf16 * 1e9), l.compulsory_bytes / (hbm * 1e6)) for l in stack.layers)
    res = {"workload": f"cfg5_resnet50_conv_stack_bf16_n{batch}", "dtype": "bf16", "layers": len(stack.layers),
           "ms_per_step": round(total, 4), "conv_ms": round(conv, 4), "maxpool_ms": round(statistics.median(pools), 4),
           "value": round(stack.flops / (total * 1e-3) / 1e12, 2), "unit": "TFLOP/s (end to end, max pool included)",
           "value_convs_only": round(stack.flops / (conv * 1e-3) / 1e12, 2),
           "sum_of_layer_rooflines_ms": round(roof_ms, 4), "frac_of_sum_roofline": round(roof_ms / conv, 3),
           "per_layer": "profiles/r01e_cfg5_layers.json (tools/time_stack.py)"}
    del stack
    torch.cuda.empty_cache()
    return res


def correctness_gate(w, xh, pf, ib, y) -> dict:
    """Sampled output pixels of the benchmarked batch vs the oracle."""
    from oracle import conv as oconv

    oh, ow = w.out_hw
    n = y.shape.n
    pixels = n * oh * ow
    idx = np.unique(np.random.default_rng(1).integers(0, pixels, 512))
    xr, wr = oconv.bf16_round(xh), oconv.bf16_round(w.filter_host())
    ref = oconv.indirect_conv_f32(xr, np.zeros(w.in_shape.c, np.float32), ib.offsets_host(), w.params, wr, None,
                                  n, oh, ow, pixel_index=idx)
    got = y.numpy().reshape(pixels, -1)[idx]
    rel = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
    ok = rel <= 1e-2
    if not ok:
        raise SystemExit(f"correctness gate failed: normwise rel error {rel:.3e} > 1e-2")
    return {"pixels_checked": int(len(idx)), "normwise_rel_err": rel, "tol": 1e-2, "pass": ok}


def reference_arm(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    r = cpu_reference(args.config, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference",
        "metric": "conv TFLOP/s (2*N*Ho*Wo*K*R*S*C / s)",
        "value": r["value"], "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (bf16-rounded operands; reference contract)", "data": "synthetic (seeded numpy)",
        "config": {"workload": w.name, "batch_per_gpu": w.in_shape.n, "parallelism": "host cores"},
        "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": r["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["icv", "reference"], default="icv")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--mr", type=int, default=128)
    ap.add_argument("--ib", choices=["per-image", "canonical"], default="per-image",
                    help="indirection-buffer form the kernels read (DESIGN.md §3)")
    ap.add_argument("--no-other", action="store_true", help="skip the per-config extra measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="image chunks pipelined in the e2e leg")
    ap.add_argument("--no-gate", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_bench(args)


if __name__ == "__main__":
    main()
