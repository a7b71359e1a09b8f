"""Benchmark of the indirect-convolution hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl icv|reference]
                    [--config cfg5|cfg1|cfg2|cfg3a|cfg3b|cfg4] [--scaling strong|weak]

One "step" = one pass of the hot path over one batch of the BASELINE
workload, every indirection buffer and packed filter built beforehand (as
the reference harness does, bench.py:156-161).  Default workload: cfg5,
BASELINE.json configs[4] -- the 53-layer ResNet-50 conv stack at N=256, the
largest configuration and the one BASELINE's "1/2/4/8 GPU" metric is about
(its `metric` quotes no single config); a step is all 53 convolutions plus
the stem's max pool, chained through the public indirect_conv API.  The
other configs (cfg1-cfg4) are reported under `other_configs`, each with its
own roofline, output gate and CPU sample.

Multi-GPU (one process per GPU, NCCL): `--gpus N` without torchrun
re-launches itself under `torch.distributed.run` (and fails loudly when the
box has fewer than N GPUs).  The batch dimension is sharded: by default the
global batch is fixed and split into contiguous image slices (strong
scaling: cfg5 256 -> 128/64/32 images per GPU);
`--scaling weak` keeps the BASELINE batch per GPU.  Filters are packed on
rank 0 and replicated by one NCCL broadcast (icv_nccl_broadcast, the only
collective; setup, outside the timed region).  Timing: CUDA events around
every step on the launching stream, L2 flushed between steps (outside the
events), barrier before, max over ranks.

`--impl reference` times the reference's own CPU algorithm for the path (the
numpy port in oracle/ of convbench's indirect_conv; the reference itself is
pure Python and cannot travel to the GPU box) on the host cores, rank 0
only, on a bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "conv TFLOP/s (2*N*Ho*Wo*K*R*S*C / s)"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "which": "fallback"}
CONV_CONFIGS = ("cfg1", "cfg2", "cfg3a", "cfg3b", "cfg4")


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        p["which"] = "measured (MEASURED_PEAKS.json)"
    except OSError:
        p = dict(PEAKS_FALLBACK)
        p["which"] = "fallback (B200_PROFILING.md)"
    try:   # int8 / fp32 peaks measured on a B200 of this pool by tools/measure_peaks.py (library GEMMs)
        with open(os.path.join(ROOT, "profiles", "peaks_extra.json")) as f:
            extra = json.load(f)
        p["int8_tops"] = extra.get("int8_tops")
        p["fp32_tflops"] = extra.get("fp32_tflops")
    except (OSError, ValueError):
        pass
    return p


def nearest_rank(sorted_values: list[float], q: float) -> float:
    """Quantile by nearest rank, element int(q * n) (reference bench.py:83-88)."""
    n = len(sorted_values)
    return sorted_values[min(int(q * n), n - 1)]


def quantiles(xs: list[float]) -> dict:
    s = sorted(xs)
    return {"median": nearest_rank(s, 0.5), "q20": nearest_rank(s, 0.2), "q80": nearest_rank(s, 0.8)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms (NVML) while running."""

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


def _oracle_conv(w, x, wt, offs, n, oh, ow):
    """One convolution of workload `w` through the oracle port (restates
    convbench.indirect.indirect_conv; uint8 through oracle/quant.py)."""
    from oracle import conv as oconv

    s = w.in_shape
    if w.dtype == "u8":
        from oracle import quant as oq
        q = w.quant
        return oq.indirect_conv_u8(x, np.full(s.c, q.input_zero_point, np.uint8), offs, w.params, wt, w.bias_host(),
                                   n, oh, ow, q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                                   q.output_zero_point, q.output_scale)
    return oconv.indirect_conv_f32(x, np.zeros(s.c, np.float32), offs, w.params, wt, w.bias_host(), n, oh, ow)


def _cpu_conv_worker(args):
    """Images [lo, hi) of conv workload `name` through the oracle port in this
    process.  Returns seconds spent in the convolution only (IB built
    outside timing, reference bench.py:156-161)."""
    name, lo, hi = args
    _init_worker()
    from oracle import conv as oconv
    from oracle import ib as oib
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    s = w.in_shape
    oh, ow = w.out_hw
    x = w.input_host(lo, hi)
    wt = w.filter_host()
    if w.dtype == "bf16":
        x, wt = oconv.bf16_round(x), oconv.bf16_round(wt)
    n = hi - lo
    offs = oib.compute_offsets((n, s.h, s.w, s.c), w.params, oh, ow, n, 4)
    t0 = time.perf_counter()
    _oracle_conv(w, x, wt, offs, n, oh, ow)
    return time.perf_counter() - t0


def _cpu_stack_worker(args):
    """cfg5 on the CPU: image `img` of the network input through the oracle
    port, layer by layer (only the layers j with j % stride == phase; the
    stem's max pool between).  Returns (seconds in the convolutions, FLOPs)."""
    img, phase, stride = args
    _init_worker()
    from oracle import conv as oconv
    from oracle import ib as oib
    from paper_1907_02129_b200.stack import stack_input_host, stack_weights_host
    from paper_1907_02129_b200.workloads import resnet50_layers

    layers = resnet50_layers(1)
    x0 = oconv.bf16_round(stack_input_host(img, img + 1))
    secs, flops = 0.0, 0
    rng = np.random.default_rng(img)
    for idx, (name, shape, p) in enumerate(layers):
        if idx % stride != phase:
            continue
        wt = oconv.bf16_round(stack_weights_host(idx, p))
        oh, ow = oib.out_hw(p, shape.h, shape.w)
        offs = oib.compute_offsets((1, shape.h, shape.w, shape.c), p, oh, ow, 1, 4)
        x = x0 if idx == 0 else oconv.bf16_round(rng.standard_normal(shape.numel, dtype=np.float32))
        t0 = time.perf_counter()
        oconv.indirect_conv_f32(x, np.zeros(shape.c, np.float32), offs, p, wt, None, 1, oh, ow)
        secs += time.perf_counter() - t0
        flops += 2 * oh * ow * p.out_channels * p.kernel_elems * p.in_channels
    return secs, flops


def _pool(procs):
    import multiprocessing as mp

    return mp.get_context("spawn").Pool(procs, initializer=_init_worker)


def cpu_conv_baseline(name: str, reps: int = 3, cores: int | None = None, single_images: int = 4) -> dict:
    """Reference algorithm on the host cores for conv workload `name`:
    leg (ii) -- one image per worker process, all cores (cache-resident
    accumulators), `reps` rounds, nearest-rank median/q20/q80 of the
    per-round throughput; leg (i) -- one process over a `single_images`
    batch, as the reference API runs a batch."""
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    cores = cores or os.cpu_count() or 1
    n_img = w.in_shape.n
    per = min(cores, n_img)
    flops_img = w.flops // n_img
    rates = []
    with _pool(per) as pool:
        pool.map(_cpu_conv_worker, [(name, 0, 1)] * per)   # warm the workers (imports)
        for r in range(reps):
            imgs = [(name, (r * per + j) % n_img, (r * per + j) % n_img + 1) for j in range(per)]
            t0 = time.perf_counter()
            pool.map(_cpu_conv_worker, imgs, chunksize=1)
            rates.append(flops_img * per / (time.perf_counter() - t0) / 1e12)
        k = min(single_images, n_img)
        t1 = pool.apply(_cpu_conv_worker, ((name, 0, k),))
    qs = quantiles(rates)
    return {"value": qs["median"], "unit": "TFLOP/s", "cores": per, "kind": "port", "cpu": cpu_model(),
            "q20": qs["q20"], "q80": qs["q80"],
            "sample": f"leg (ii): {per} images of {name} per round, one per worker process (OMP_NUM_THREADS=1), "
                      f"{reps} rounds, wall clock, nearest-rank median; IB built outside timing",
            "single_process": {"value": flops_img * k / t1 / 1e12, "unit": "TFLOP/s", "cores": 1,
                               "sample": f"leg (i): one process, a batch of {k} images through one call"}}


def cpu_stack_baseline(cores: int | None = None, reps: int = 1) -> dict:
    """cfg5 on the host cores: each worker process runs one image through
    all 53 layers (reps rounds)."""
    cores = cores or os.cpu_count() or 1
    per = min(cores, 16)
    rates = []
    with _pool(per) as pool:
        for r in range(reps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_stack_worker, [(r * per + j, 0, 1) for j in range(per)], chunksize=1)
            wall = time.perf_counter() - t0
            rates.append(sum(f for _, f in res) / wall / 1e12)
    qs = quantiles(rates)
    return {"value": qs["median"], "unit": "TFLOP/s", "cores": per, "kind": "port", "cpu": cpu_model(),
            "q20": qs["q20"], "q80": qs["q80"],
            "sample": f"{per} images of cfg5, one per worker process (OMP_NUM_THREADS=1), each through all 53 "
                      f"convolutions (8.17 GFLOP per image), {reps} round(s), wall clock incl. per-layer setup"}


def cpu_reference_steps(name: str, steps: int, warmup: int) -> tuple[list[float], dict]:
    """Per-step throughputs (TFLOP/s) of the reference algorithm on the host
    cores, each step a bounded sample: cfg5 -- one image per worker through
    every 4th layer of the stack (phase = step mod 4, ~2.5 s); conv configs
    -- one image per worker."""
    cores = os.cpu_count() or 1
    rates = []
    if name == "cfg5":
        per = min(cores, 16)
        with _pool(per) as pool:
            for it in range(warmup + steps):
                t0 = time.perf_counter()
                res = pool.map(_cpu_stack_worker, [(it * per + j, it % 4, 4) for j in range(per)], chunksize=1)
                wall = time.perf_counter() - t0
                if it >= warmup:
                    rates.append(sum(f for _, f in res) / wall / 1e12)
        sample = (f"{per} images of cfg5 per step, one per worker process (OMP_NUM_THREADS=1), each through every "
                  "4th layer of the stack (phase = step mod 4), wall clock")
        return rates, {"cores": per, "sample": sample}
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    n_img = w.in_shape.n
    per = min(cores, n_img)
    flops_img = w.flops // n_img
    with _pool(per) as pool:
        for it in range(warmup + steps):
            imgs = [(name, (it * per + j) % n_img, (it * per + j) % n_img + 1) for j in range(per)]
            t0 = time.perf_counter()
            pool.map(_cpu_conv_worker, imgs, chunksize=1)
            if it >= warmup:
                rates.append(flops_img * per / (time.perf_counter() - t0) / 1e12)
    return rates, {"cores": per, "sample": f"{per} images of {name} per step, one per worker process, wall clock"}


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    rates, meta = cpu_reference_steps(args.config, args.steps, args.warmup)
    qs = quantiles(rates)
    value = statistics.mean(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32 (bf16-rounded operands; the reference contract)", "data": "synthetic (seeded numpy)",
        "config": {"workload": workload_name(args.config), "parallelism": "host cores (rank 0 only)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": meta["cores"], "kind": "port", "cpu": cpu_model(),
                         "median": qs["median"], "q20": qs["q20"], "q80": qs["q80"], "sample": meta["sample"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm helpers
def workload_name(name: str) -> str:
    if name == "cfg5":
        return "cfg5_resnet50_conv_stack_bf16_n256"
    from paper_1907_02129_b200.workloads import CONFIGS
    return CONFIGS[name].name


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


def peak_for(dtype: str, bound: str, peaks: dict) -> tuple[float, str, str]:
    """(peak, unit, source) of the roofline denominator."""
    if bound == "hbm":
        return peaks["hbm_gbs"], "GB/s", peaks["which"] + " hbm_gbs"
    if dtype == "u8":
        if peaks.get("int8_tops"):
            return peaks["int8_tops"], "TOP/s", "int8 GEMM measured on a pool B200 (profiles/peaks_extra.json)"
        return 2 * peaks["bf16_tflops"], "TOP/s", "2x bf16 (nominal ratio; int8 peak unmeasured)"
    if dtype == "f32":
        if peaks.get("fp32_tflops"):
            return peaks["fp32_tflops"], "TFLOP/s", "fp32 CUDA-core GEMM measured on a pool B200 (profiles/peaks_extra.json)"
        return 75.0, "TFLOP/s", "nominal fp32 CUDA-core peak"
    return peaks["bf16_tflops"], "TFLOP/s", peaks["which"] + " bf16_tflops (burst)"


def roofline_of(dtype: str, flops: float, nbytes: float, ms: float, peaks: dict) -> dict:
    """Roofline of one kernel launch.  The bound is the one with the larger
    minimum time: FLOPs over the dtype's compute peak (bf16 / int8 tensor
    pipe; cfg1's exact f32 runs on the CUDA cores) vs algorithmic bytes over
    HBM bandwidth."""
    cpk, cunit, csrc = peak_for(dtype, "tensor", peaks)
    t_compute = flops / (cpk * 1e12)
    t_hbm = nbytes / (peaks["hbm_gbs"] * 1e9)
    if t_compute >= t_hbm:
        achieved = flops / (ms * 1e-3) / 1e12
        return {"bound": "tensor" if dtype != "f32" else "fp32_core", "achieved": round(achieved, 2), "peak": cpk,
                "unit": cunit, "frac": round(achieved / cpk, 4), "peak_source": csrc}
    achieved = nbytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / peaks["hbm_gbs"], 4), "peak_source": peaks["which"] + " hbm_gbs"}


def load_traffic(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            entry = json.load(f).get(key)
        return None if entry is None else entry["bytes"]
    except (OSError, ValueError, KeyError):
        return None


def setup_problem(name: str, n_lo: int, n_hi: int, device, replicate=None, mr: int = 128, per_image: bool = True,
                  rank: int = 0):
    """Upload images [n_lo, n_hi) of conv workload `name`, build the IB on
    the device, pack the filter on rank 0 and replicate it (or pack locally
    when `replicate` is None)."""
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
    bias_t = None if bias is None else torch.from_numpy(bias)
    if replicate is None:
        filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                                torch.from_numpy(w.filter_host()).to(device).to(dt))
        pf = icv.pack_filter(filt, bias_t, p, tile, quant=qp)
    else:
        filt = None
        if rank == 0:
            filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                                    torch.from_numpy(w.filter_host()).to(device).to(dt))
        pf = replicate(filt, bias_t, p, tile, dt, qp)
    zero = icv.make_zero_row(p.in_channels, dtype=dt, device=device, fill=zero_fill)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, per_image=per_image)
    y = icv.NhwcTensor.empty(out_shape, dtype=dt, device=device)
    return w, x, xh, pf, ib, y, tile


def conv_gate(w, xh, ib, y, n_lo: int = 0, pixels: int = 512) -> dict:
    """The benchmarked output of a conv workload vs the oracle on sampled
    pixels (reference bench.py:124-142 gate protocol): float32 and uint8
    bit-exact, bf16 within BASELINE's rel 1e-2 (normwise)."""
    from oracle import conv as oconv
    from oracle import quant as oq

    oh, ow = w.out_hw
    n = y.shape.n
    total = n * oh * ow
    idx = np.unique(np.random.default_rng(1).integers(0, total, min(pixels, total)))
    offs = ib.offsets_host()
    k = w.params.out_channels
    got = y.numpy().reshape(total, k)[idx]
    if w.dtype == "u8":
        q = w.quant
        ref = oq.indirect_conv_u8(xh, np.full(w.in_shape.c, q.input_zero_point, np.uint8), offs, w.params,
                                  w.filter_host(), w.bias_host(), n, oh, ow, q.input_zero_point, q.input_scale,
                                  q.kernel_zero_point, q.kernel_scale, q.output_zero_point, q.output_scale,
                                  pixel_index=idx)
        ok = bool(np.array_equal(got, ref))
        res = {"pixels_checked": int(len(idx)), "mismatches": int((got != ref).sum()), "rule": "bit-exact",
               "pass": ok}
    elif w.dtype == "f32":
        ref = oconv.indirect_conv_f32(xh, np.zeros(w.in_shape.c, np.float32), offs, w.params, w.filter_host(),
                                      w.bias_host(), n, oh, ow, pixel_index=idx)
        ok = got.tobytes() == ref.tobytes()
        res = {"pixels_checked": int(len(idx)), "rule": "bit-exact", "pass": ok}
    else:
        ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(w.in_shape.c, np.float32), offs, w.params,
                                      oconv.bf16_round(w.filter_host()), w.bias_host(), n, oh, ow, pixel_index=idx)
        rel = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
        ok = rel <= 1e-2
        res = {"pixels_checked": int(len(idx)), "normwise_rel_err": rel, "rule": "normwise rel <= 1e-2", "pass": ok}
    if not ok:
        raise SystemExit(f"correctness gate failed on {w.name}: {res}")
    return res


def stack_gate(stack, layer_names=("stem", "s1b1_1x1a", "s1b1_3x3", "s2b1_3x3", "s2b1_proj", "s3b2_3x3",
                                   "s4b1_3x3", "s4b3_1x1b"), pixels: int = 96) -> dict:
    """cfg5 gate: for a set of layers spanning every kernel family, sampled
    output pixels of the benchmarked pass vs the oracle on that layer's
    actual bf16 input (parity per layer on its own input)."""
    from oracle import conv as oconv

    worst = 0.0
    checked = []
    for layer in stack.layers:
        if layer.name not in layer_names:
            continue
        s, o = layer.input.shape, layer.output.shape
        total = o.n * o.h * o.w
        idx = np.unique(np.random.default_rng(layer.index).integers(0, total, pixels))
        xh = layer.input.numpy()
        ref = oconv.indirect_conv_f32(xh, np.zeros(s.c, np.float32), layer.ib.offsets_host(), layer.params,
                                      layer.weights_host, None, o.n, o.h, o.w, pixel_index=idx)
        got = layer.output.numpy().reshape(total, -1)[idx]
        rel = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
        worst = max(worst, rel)
        checked.append(layer.name)
    ok = worst <= 1e-2
    res = {"layers_checked": checked, "pixels_per_layer": pixels, "worst_normwise_rel_err": worst,
           "rule": "normwise rel <= 1e-2 per layer", "pass": ok}
    if not ok:
        raise SystemExit(f"correctness gate failed on cfg5: {res}")
    return res


# ---------------------------------------------------------------- headline: cfg5 stack
def stack_layer_table(stack, peaks: dict, passes: int = 3) -> list[dict]:
    """Per-layer median CUDA-event times of `passes` whole-stack passes."""
    import torch

    from paper_1907_02129_b200 import _lib

    per = []
    for _ in range(passes):
        _, _, layers = stack.timed_run()
        per.append(layers)
    rows = []
    for i, layer in enumerate(stack.layers):
        ms = statistics.median(p[i] for p in per)
        r = roofline_of("bf16", layer.flops, layer.compulsory_bytes, ms, peaks)
        t_roof = max(layer.flops / (peaks["bf16_tflops"] * 1e12), layer.compulsory_bytes / (peaks["hbm_gbs"] * 1e9))
        rows.append({"layer": layer.name,
                     "kernel": _lib.kernel_name(layer.params, layer.input.shape, torch.bfloat16),
                     "us": round(ms * 1e3, 2), "tflops": round(layer.flops / (ms * 1e-3) / 1e12, 1),
                     "roofline_us": round(t_roof * 1e6, 2), "frac": r["frac"], "bound": r["bound"],
                     "flops": layer.flops, "bytes": layer.compulsory_bytes})
    return rows


def dominant_roofline(rows: list[dict], peaks: dict) -> dict:
    """Roofline of the step's dominant kernel: the (kernel, bound) class with
    the largest share of the step's conv time; achieved = its algorithmic
    bytes (HBM-bound class) or FLOPs (tensor-bound class) summed over its
    launches / its summed launch time."""
    # (one class per kernel family: the dense-A kernel's single-CTA and CTA-pair
    # plans are the same __global__ template, like its BLOCK_N variants)
    groups: dict[tuple[str, str], list[dict]] = {}
    for r in rows:
        groups.setdefault((r["kernel"].replace(",pair>", ">"), r["bound"]), []).append(r)
    total_us = sum(r["us"] for r in rows)
    (kern, bound), members = max(groups.items(), key=lambda kv: sum(r["us"] for r in kv[1]))
    us = sum(r["us"] for r in members)
    if bound == "hbm":
        achieved = sum(r["bytes"] for r in members) / (us * 1e-6) / 1e9
        peak, unit = peaks["hbm_gbs"], "GB/s"
    else:
        achieved = sum(r["flops"] for r in members) / (us * 1e-6) / 1e12
        peak, unit = peaks["bf16_tflops"], "TFLOP/s"
    traffic = load_traffic(f"cfg5:{kern}:{bound}")
    return {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": kern, "launches_per_step": len(members),
            "share_of_conv_time": round(us / total_us, 3),
            "plans": {k: sum(1 for r in members if r["kernel"] == k) for k in sorted({r["kernel"] for r in members})},
            "layers": [r["layer"] for r in members],
            "per_launch": "algorithmic bytes (input + filter + output) or FLOPs of each launch / its CUDA-event time, "
                          "summed over the class",
            "peak_source": peaks["which"]}


class StackE2E:
    """cfg5 end to end through the public API with host buffers: the shard
    is cut into `chunks` image chunks, each with its own stack (activations,
    per-image IBs bound to that chunk's input buffer, replicated packed
    filters); per step every chunk's input goes pinned host -> device, its
    53 indirect_conv calls (+ max pool) are issued from Python (no graph
    replay), and its final activation goes device -> pinned host; chunk i's
    H2D overlaps chunk i-1's convolutions and chunk i-2's D2H on three
    streams."""

    def __init__(self, lo: int, hi: int, chunks: int, device, replicate=None):
        import torch

        from paper_1907_02129_b200.stack import IMAGE_ELEMS, ResNet50Stack, stack_input_host

        self.device = device
        n = hi - lo
        chunks = max(1, min(chunks, n))
        bounds = [lo + n * i // chunks for i in range(chunks + 1)]
        self.stacks = [ResNet50Stack(device=device, images=(bounds[i], bounds[i + 1]), replicate=replicate)
                       for i in range(chunks)]
        xh = stack_input_host(lo, hi)
        self.x_pinned = torch.from_numpy(xh).to(torch.bfloat16).pin_memory()
        self.offsets = [(b - lo) * IMAGE_ELEMS for b in bounds]
        last = self.stacks[0].layers[-1].output
        per_img_out = last.shape.h * last.shape.w * last.shape.c
        self.y_pinned = torch.empty(n * per_img_out, dtype=torch.bfloat16).pin_memory()
        self.out_offsets = [(b - lo) * per_img_out for b in bounds]
        self.h2d_bytes = int(self.x_pinned.numel() * 2)
        self.d2h_bytes = int(self.y_pinned.numel() * 2)
        self.s_h2d, self.s_cmp, self.s_d2h = (torch.cuda.Stream(device) for _ in range(3))
        self.flops = sum(s.flops for s in self.stacks)

    def step(self):
        import torch

        cur = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(cur)
        for st in (self.s_h2d, self.s_cmp, self.s_d2h):
            st.wait_event(start)
        for i, stack in enumerate(self.stacks):
            a, b = self.offsets[i], self.offsets[i + 1]
            with torch.cuda.stream(self.s_h2d):
                stack.input.data.copy_(self.x_pinned[a:b], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.s_h2d)
            self.s_cmp.wait_event(ev_in)
            with torch.cuda.stream(self.s_cmp):
                stack.run()
                ev_out = torch.cuda.Event()
                ev_out.record(self.s_cmp)
            self.s_d2h.wait_event(ev_out)
            with torch.cuda.stream(self.s_d2h):
                oa, ob = self.out_offsets[i], self.out_offsets[i + 1]
                self.y_pinned[oa:ob].copy_(stack.layers[-1].output.data, non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.s_d2h)
        cur.wait_event(done)


def replicator(comm, rank: int, world: int, device):
    """Filter replication hooks for the data-parallel runs: rank 0 packs,
    one NCCL broadcast per packed filter (the operator's only collective)."""
    import paper_1907_02129_b200 as icv

    def stack_hook(pf):
        if world > 1:
            icv.broadcast_packed_filter(pf, 0, comm=comm)

    def conv_hook(filt, bias, params, tile, dt, qp):
        return icv.replicate_filter(filt, bias, params, tile, rank=rank, device=device, compute_dtype=dt, quant=qp,
                                    comm=comm if world > 1 else None) if world > 1 else \
            icv.pack_filter(filt, bias, params, tile, quant=qp)

    return stack_hook, conv_hook


def bench_stack(args, ctx) -> dict:
    """Headline cfg5: the whole stack per step on this rank's shard."""
    import torch

    from paper_1907_02129_b200 import _lib
    from paper_1907_02129_b200.dist import shard_range
    from paper_1907_02129_b200.stack import ResNet50Stack

    world, rank, device = ctx["world"], ctx["rank"], ctx["device"]
    gbatch = 256 if args.scaling == "strong" else 256 * world
    lo, hi = shard_range(gbatch, world, rank)
    stack = ResNet50Stack(device=device, images=(lo, hi), replicate=ctx["stack_hook"])
    flush = ctx["flush"]
    # the device-timed step replays the pass as one CUDA graph (the e2e leg
    # below issues every indirect_conv call from Python instead)
    step = stack.run if args.no_graph else stack.graphed()
    res = run_timed(args, ctx, step, flush, None if args.no_graph else stack.graph_launches)
    res["cuda_graph"] = not args.no_graph
    res.update({"flops_rank": stack.flops, "global_batch": gbatch, "batch_rank": hi - lo})
    if rank == 0:
        rows = stack_layer_table(stack, ctx["peaks"])
        res["layers"] = rows
        res["roofline"] = dominant_roofline(rows, ctx["peaks"])
        t_roof = sum(r["roofline_us"] for r in rows)
        t_meas = sum(r["us"] for r in rows)
        res["stack_roofline"] = {"sum_layer_roofline_us": round(t_roof, 1), "sum_layer_measured_us": round(t_meas, 1),
                                 "frac": round(t_roof / t_meas, 4),
                                 "rule": "per layer max(FLOPs / bf16 peak, compulsory bytes / HBM BW), summed"}
        res["gate"] = None if args.no_gate else stack_gate(stack)
        res["conv_kernels"] = sorted({r["kernel"] for r in rows})
    del stack
    torch.cuda.empty_cache()
    e2e = StackE2E(lo, hi, args.e2e_chunks, device, replicate=ctx["stack_hook"])
    res["e2e"] = run_e2e(args, ctx, e2e.step, e2e.flops, e2e.h2d_bytes, e2e.d2h_bytes,
                         f"pinned host input -> device, per chunk of {len(e2e.stacks)} the 53 indirect_conv calls "
                         "(+ max pool) issued from Python (no graph), final activation -> pinned host; "
                         "H2D / compute / D2H of successive chunks overlap on three streams")
    res["e2e"]["chunks"] = len(e2e.stacks)
    del e2e
    torch.cuda.empty_cache()
    res["conv_kernel"] = "53 launches: " + ", ".join(res.get("conv_kernels", []))
    return res


def run_timed(args, ctx, fn, flush, launches_per_replay: int | None = None) -> dict:
    """K timed steps after W warm-ups, barrier + synchronize on both sides;
    the per-rank total is max-reduced over ranks.  `launches_per_replay`:
    fn replays a CUDA graph holding that many libicv kernels (the host-side
    launch counter does not see replays)."""
    import torch
    import torch.distributed as dist

    from paper_1907_02129_b200 import _lib

    world, sampler = ctx["world"], ctx["sampler"]
    for _ in range(args.warmup):
        flush()
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    if sampler:
        sampler.mark("t0")
    times = time_steps(fn, args.steps, 0, flush)
    if sampler:
        sampler.mark("t1")
    launches = _lib.launch_count() - l0
    if launches_per_replay is not None:
        launches += launches_per_replay * args.steps
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=ctx["device"])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    return {"times": times, "total_ms": total, "launches": launches}


def run_e2e(args, ctx, fn, flops_rank: int, h2d: int, d2h: int, path: str) -> dict:
    import torch
    import torch.distributed as dist

    world = ctx["world"]
    steps = max(3, min(args.steps, 20))
    for _ in range(max(args.warmup, 3)):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = time_steps(fn, steps, 0, ctx["flush"])
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=ctx["device"])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return {"value": round(flops_rank * world * steps / (total * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
            "ms_per_step": round(total / steps, 4), "cuda_graph": False, "path": path}


# ---------------------------------------------------------------- conv configs
def bench_conv(args, ctx, name: str) -> dict:
    """Headline for a conv config (--config cfgN): its batch per step."""
    import torch

    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200 import _lib
    from paper_1907_02129_b200.dist import shard_range
    from paper_1907_02129_b200.workloads import CONFIGS

    world, rank, device = ctx["world"], ctx["rank"], ctx["device"]
    w0 = CONFIGS[name]
    gbatch = w0.in_shape.n if args.scaling == "strong" else w0.in_shape.n * world
    if gbatch < world:
        raise SystemExit(f"{name}: a global batch of {gbatch} cannot be sharded over {world} GPUs")
    import paper_1907_02129_b200.workloads as wl
    wl.CONFIGS["_bench"] = w0.with_batch(gbatch)
    lo, hi = shard_range(gbatch, world, rank)
    w, x, xh, pf, ib, y, tile = setup_problem("_bench", lo, hi, device, ctx["conv_hook"], per_image=args.ib == "per-image",
                                              rank=rank)
    res = run_timed(args, ctx, lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y), ctx["flush"])
    wl_rank = w0.with_batch(hi - lo)
    res.update({"flops_rank": wl_rank.flops, "global_batch": gbatch, "batch_rank": hi - lo})
    if rank == 0:
        ms = statistics.mean(res["times"])
        res["roofline"] = roofline_of(w0.dtype, wl_rank.flops, wl_rank.compulsory_bytes, ms, ctx["peaks"])
        res["roofline"]["traffic"] = load_traffic(w0.name)
        res["gate"] = None if args.no_gate else conv_gate(wl_rank, xh, ib, y)
        res["conv_kernel"] = _lib.kernel_name(w0.params, w0.in_shape, x.dtype)
    # e2e: pinned host input -> device, the API call, output -> pinned host
    dt = x.dtype
    x_pinned = torch.from_numpy(xh).to(dt).pin_memory()
    y_pinned = torch.empty(y.data.numel(), dtype=dt).pin_memory()

    def e2e_step():
        x.data.copy_(x_pinned, non_blocking=True)
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
        y_pinned.copy_(y.data, non_blocking=True)

    res["e2e"] = run_e2e(args, ctx, e2e_step, wl_rank.flops, x_pinned.numel() * x_pinned.element_size(),
                         y_pinned.numel() * y_pinned.element_size(),
                         "pinned host input -> device, one indirect_conv call (Python API, no graph), output -> pinned "
                         "host, all on the current stream")
    return res


def other_config(name: str, ctx, args) -> dict:
    """A BASELINE conv config measured on one GPU: the default kernel and the
    IB-gather kernel (algorithm="gather": the paper's mainloop) when they
    differ, rooflines, output gate, CPU sample."""
    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200 import _lib
    from paper_1907_02129_b200.workloads import CONFIGS

    device, peaks, flush = ctx["device"], ctx["peaks"], ctx["flush"]
    w0 = CONFIGS[name]
    w, x, xh, pf, ib, y, tile = setup_problem(name, 0, w0.in_shape.n, device, per_image=args.ib == "per-image")
    reps = max(10, args.steps // 5)
    out = {"workload": w.name, "dtype": w.dtype}
    legs = {"auto": "auto"}
    k_auto = _lib.kernel_name(w.params, w.in_shape, x.dtype)
    flags_g = icv.indirect.conv_flags(ib, pf, x.dtype, "gather")
    k_gather = _lib.kernel_name(w.params, w.in_shape, x.dtype, flags_g)
    if k_gather != k_auto:
        legs["gather"] = "gather"
    for leg, alg in legs.items():
        t = time_steps(lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y, algorithm=alg), reps, 3, flush)
        qs = quantiles(t)
        ms = qs["median"]
        entry = {"kernel": k_auto if leg == "auto" else k_gather, "ms_per_step": round(ms, 5),
                 "ms_q20": round(qs["q20"], 5), "ms_q80": round(qs["q80"], 5),
                 "value": round(w.flops / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s" if w.dtype != "u8" else "TOP/s",
                 "roofline": roofline_of(w.dtype, w.flops, w.compulsory_bytes, ms, peaks),
                 "gate": None if args.no_gate else conv_gate(w, xh, ib, y)}
        entry["roofline"]["traffic"] = load_traffic(w.name if leg == "auto" else f"{w.name}:gather")
        if leg == "auto":
            out.update(entry)
        else:
            out["ib_gather_kernel"] = entry
    if not args.no_cpu:
        out["cpu_baseline"] = cpu_conv_baseline(name, reps=2)
    if not w.params.is_pointwise_unit_stride() and name in ("cfg2", "cfg4"):
        out["im2col_gemm"] = gemm_baseline(w, x, pf, tile, flush, reps, peaks)
        out["im2col_gemm"]["indirect_speedup"] = round(out["im2col_gemm"]["ms_per_step"] / out["ms_per_step"], 3)
    return out


def gemm_baseline(w, x, pf, tile, flush, reps: int, peaks: dict) -> dict:
    """The paper's comparison (§2.1): the GEMM-based variant --
    im2row patch matrix written to HBM, then a dense TMA-tiled tcgen05 GEMM
    over it (the patch matrix as a 1 x P image of R*S*C channels: the
    dense-A kernel, no indirection) -- both inside every step, as the
    reference's gemm_conv does (im2col.py:117-131).  Also the GEMM alone."""
    import torch

    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200 import _lib

    pm = icv.build_patch_matrix(x, w.params)
    icv.gemm_only(pm, pf, tile)

    def gemm_step():
        icv.build_patch_matrix(x, w.params, out=pm)
        icv.gemm_only(pm, pf, tile)

    ms = quantiles(time_steps(gemm_step, reps, 3, flush))["median"]
    ms_gemm = quantiles(time_steps(lambda: icv.gemm_only(pm, pf, tile), reps, 3, flush))["median"]
    eb = pm.matrix.element_size()
    gemm_bytes = pm.rows * pm.cols * eb + w.params.out_channels * pm.cols * eb + pm.rows * w.params.out_channels * eb
    p1 = icv.ConvParams(1, 1, in_channels=pm.cols, out_channels=pf.k_out)
    res = {"ms_per_step": round(ms, 5), "value": round(w.flops / (ms * 1e-3) / 1e12, 2),
           "kernels": ["icv_im2col", _lib.kernel_name(p1, icv.Shape4(1, 1, pm.rows, pm.cols), x.dtype)],
           "patch_matrix_mb": round(pm.allocated_bytes / 1e6, 2),
           "gemm_only_ms": round(ms_gemm, 5),
           "gemm_only_roofline": roofline_of(w.dtype, w.flops, gemm_bytes, ms_gemm, peaks),
           "note": "reference im2col.py gemm_conv: patch matrix rebuilt every step, then the dense GEMM"}
    del pm
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- driver
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args) -> int:
    """`--gpus N` without torchrun: re-launch this script as N ranks under
    torch.distributed.run (NCCL_DEBUG=INFO so each communicator's rank count
    is logged); fail loudly when the box has fewer than N GPUs."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but this box has {have} GPU(s)",
                          "n_gpus": args.gpus}), flush=True)
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, found {have}", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def gpu_bench(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    comm = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=device)
        from paper_1907_02129_b200.dist import NcclComm

        comm = NcclComm.from_process_group(device)
        print(f"bench.py rank {rank}: icv NCCL communicator of {comm.size()} ranks on {device}", file=sys.stderr,
              flush=True)
    stack_hook, conv_hook = replicator(comm, rank, world, device)
    peaks = load_peaks()
    sampler = ClockSampler(local).start() if rank == 0 else None
    ctx = {"world": world, "rank": rank, "device": device, "peaks": peaks, "flush": make_l2_flush(device),
           "sampler": sampler, "stack_hook": stack_hook, "conv_hook": conv_hook, "comm": comm}
    name = args.config
    head = bench_stack(args, ctx) if name == "cfg5" else bench_conv(args, ctx, name)
    clocks = sampler.stop(("t0", "t1")) if sampler else None

    other = {}
    cpu = None
    if rank == 0 and world == 1 and not args.no_other:
        for oname in CONV_CONFIGS:
            if oname != name:
                other[oname] = other_config(oname, ctx, args)
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_stack_baseline() if name == "cfg5" else cpu_conv_baseline(name)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return
    total_ms = head["total_ms"]
    # FLOPs are linear in the batch: the whole job's FLOPs per step are the
    # global batch's (rank shards differ by at most one image)
    flops_total = head["flops_rank"] / head["batch_rank"] * head["global_batch"] * args.steps
    value = flops_total / (total_ms * 1e-3) / 1e12
    qs = quantiles(head["times"])
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 6),
        "ms_per_step_median": round(qs["median"], 6),
        "ms_per_step_q20": round(qs["q20"], 6),
        "ms_per_step_q80": round(qs["q80"], 6),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "bf16" if name not in ("cfg1", "cfg4") else {"cfg1": "f32", "cfg4": "u8"}[name],
        "data": "synthetic (seeded numpy; BASELINE configs are synthetic)",
        "config": {"workload": workload_name(name), "global_batch": head["global_batch"],
                   "batch_per_gpu_rank0": head["batch_rank"], "parallelism": f"dp{world} (batch-sharded, "
                   f"{'fixed global batch' if args.scaling == 'strong' else 'fixed batch per GPU'})",
                   "mr": 128, "index_dtype": "int64", "ib_layout": args.ib,
                   "l2": "flushed between steps (256 MiB device write + 256 MiB read, outside the timed events)",
                   "conv_kernel": head.get("conv_kernel"), "cuda_graph": head.get("cuda_graph", False),
                   "pdl": True},
        "roofline": head.get("roofline"),
        "e2e": head["e2e"],
        "gpu_launches": int(head["launches"]),
        "clocks": clocks,
        "cpu_baseline": cpu,
        "gate": head.get("gate"),
    }
    if "stack_roofline" in head:
        line["stack_roofline"] = head["stack_roofline"]
        line["per_layer"] = [{k: r[k] for k in ("layer", "kernel", "us", "roofline_us", "frac", "bound")}
                             for r in head["layers"]]
    line["other_configs"] = other or None
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["icv", "reference"], default="icv")
    ap.add_argument("--config", default="cfg5", choices=["cfg5", *CONV_CONFIGS])
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: fixed global batch split over the GPUs (SURVEY.md §8(e)); weak: BASELINE batch per GPU")
    ap.add_argument("--ib", choices=["per-image", "canonical"], default="per-image",
                    help="indirection-buffer form the kernels read (DESIGN.md §3)")
    ap.add_argument("--no-other", action="store_true", help="skip the per-config extra measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="image chunks pipelined in the e2e leg")
    ap.add_argument("--no-gate", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="cfg5: issue the timed passes from Python, no CUDA graph")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    elif "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args))
    else:
        gpu_bench(args)


if __name__ == "__main__":
    main()
