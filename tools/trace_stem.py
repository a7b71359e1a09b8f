"""Phase breakdown of the channel-poor (stem) kernel from a debug build with
ICV_TRACE (cycles per tile, mean over CTAs):
    make -C paper_1907_02129_b200/csrc variant NAME=trace DEFS=-DICV_TRACE
    ICV_LIB=paper_1907_02129_b200/_lib/libicv_trace.so python tools/trace_stem.py cfg3a"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3a"
    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    flush.fill_(1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    e.record()
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    oh, ow = w.out_hw
    tiles = w.in_shape.n * oh * ow / 128 / 148
    tr = buf[:148].astype(np.float64) / tiles
    print(f"{name}: {s.elapsed_time(e) * 1e3:.1f} us, {tiles:.1f} tiles per CTA; cycles per tile:")
    names = ["wait window+bar", "convert+bar", "wait empty", "build+arrive", "prepare"]
    for h in range(2):
        print(f"  producer half {h}: " + ", ".join(f"{n} {tr[:, 30 + 5 * h + i].mean():.0f}" for i, n in enumerate(names)))
    print(f"  MMA: wait tmem-empty {tr[:, 26].mean():.0f}, wait full {tr[:, 27].mean():.0f}")
    print(f"  epilogue warp 0: wait {tr[:, 28].mean():.0f}, work {tr[:, 29].mean():.0f}")


if __name__ == "__main__":
    main()
