"""A/B a native plan knob on cfg5 layers (N=256, L2 flushed, median of 7).

    python tools/ab_knob.py s3b2_1x1a,s1b1_3x3 dense_pf 0,1,2 [knob2=v ...]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200.stack import ResNet50Stack  # noqa: E402


def main():
    names, knob, values = sys.argv[1].split(","), sys.argv[2], [int(v) for v in sys.argv[3].split(",")]
    for kv in sys.argv[4:]:
        k, v = kv.split("=")
        L.set_tuning(k, int(v))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    stack = ResNet50Stack(device=dev)
    flush = bench.make_l2_flush(dev)
    by = {l.name: l for l in stack.layers}
    for n in names:
        l = by[n]
        for v in values:
            L.set_tuning(knob, v)
            t = bench.time_steps(lambda: stack.run_layer(l), 7, 2, flush)
            print(f"{n:12s} {knob}={v:<4d} {L.kernel_name(l.params, l.input.shape, torch.bfloat16):32s} "
                  f"{statistics.median(t) * 1e3:8.1f} us", flush=True)


if __name__ == "__main__":
    main()
