"""Run selected layers of the cfg5 ResNet-50 stack (N=256 by default) in
isolation, for ncu captures and quick A/B timings.

    python tools/prof_stack_layers.py --layers s3b2_1x1b,s1b1_3x3 [--iters 3] [--batch 256]

The whole stack is built (IBs, packed filters, activations), then each named
layer's convolution runs `iters` times with an L2 flush before every launch;
per-layer median CUDA-event times are printed.  Under ncu use
`-k regex:igemm -c <layers * iters>`: no conv kernel launches before them.
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200.stack import ResNet50Stack  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", required=True)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    stack = ResNet50Stack(batch=args.batch, device=dev)
    by_name = {l.name: l for l in stack.layers}
    names = [n for n in args.layers.split(",") if n]
    flush = bench.make_l2_flush(dev)
    torch.cuda.synchronize()
    for n in names:
        layer = by_name[n]
        times = []
        for _ in range(args.iters):
            flush()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            stack.run_layer(layer)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        ms = statistics.median(times)
        print(f"{n:12s} {L.kernel_name(layer.params, layer.input.shape, torch.bfloat16):24s} "
              f"{ms * 1e3:8.1f} us  {layer.flops / ms / 1e9:7.1f} TFLOP/s  "
              f"{layer.compulsory_bytes / ms / 1e6:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
