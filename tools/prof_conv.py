"""Run one BASELINE config's convolution a few times (for ncu captures).

    python tools/prof_conv.py --config cfg2 --iters 5
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--mr", type=int, default=128)
    args = ap.parse_args()
    from paper_1907_02129_b200.workloads import CONFIGS

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(args.config, 0, CONFIGS[args.config].in_shape.n, dev, mr=args.mr)
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(args.iters):
        flush_l2()
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    print("done", args.config)


if __name__ == "__main__":
    main()
