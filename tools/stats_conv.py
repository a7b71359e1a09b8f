"""Per-role cycle breakdown of the tcgen05 kernel (debug build with
ICV_STATS counters).  Usage on the GPU box:

    make -C paper_1907_02129_b200/csrc stats
    ICV_LIB=$PWD/paper_1907_02129_b200/_lib/libicv_stats.so python tools/stats_conv.py --config cfg2
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402

NAMES = ["prod_empty_wait", "prod_loop", "mma_full_wait", "mma_tempty_wait", "mma_loop", "epi_tfull_wait",
         "epi_loop", "kblocks"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--mr", type=int, default=128)
    args = ap.parse_args()
    from paper_1907_02129_b200.workloads import CONFIGS

    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(args.config, 0, CONFIGS[args.config].in_shape.n, dev,
                                                    mr=args.mr)
    fn = L.lib().icv_debug_stats
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(3):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 8), np.uint64)
    fn(None, 1)
    flush_l2()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    e.record()
    torch.cuda.synchronize()
    fn(buf.ctypes.data, 0)
    sms = 148
    st = buf[:sms].astype(np.float64)
    print(f"{args.config}: {s.elapsed_time(e) * 1e3:.1f} us")
    for i, n in enumerate(NAMES):
        col = st[:, i]
        print(f"  {n:18s} mean {col.mean():10.0f}  min {col.min():10.0f}  max {col.max():10.0f}")


if __name__ == "__main__":
    main()
