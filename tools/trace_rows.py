"""Role breakdown of the row-sliding kernel (debug build with -DICV_ROWS_PHASES):
cycles per tile, mean over CTAs."""
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
    for _ in range(3):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    torch.empty(256 << 20, dtype=torch.uint8, device=dev).fill_(1)
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    oh, ow = w.out_hw
    tiles = w.in_shape.n * oh / 148
    tr = buf[:148].astype(np.float64) / tiles
    print(f"{name}: {tiles:.1f} tiles per CTA; cycles per tile")
    print(f"  loader:     wait stage_free {tr[:, 30].mean():.0f}, issue {tr[:, 32].mean():.0f}, other {tr[:, 31].mean():.0f}")
    print(f"  converters: wait mdone {tr[:, 34].mean():.0f}, wait stage_full {tr[:, 35].mean():.0f}, "
          f"convert {tr[:, 36].mean():.0f}, other {tr[:, 37].mean():.0f}")
    print(f"  MMA:        wait tmem-empty {tr[:, 38].mean():.0f}, wait rows {tr[:, 39].mean():.0f}, "
          f"MMA instructions {tr[:, 40].mean():.0f}, fence/commit/sync/other {tr[:, 41].mean():.0f}")
    print(f"  epilogue w0: wait tfull {tr[:, 42].mean():.0f}, tmem ld {tr[:, 43].mean():.0f}, "
          f"convert {tr[:, 44].mean():.0f}, stage {tr[:, 45].mean():.0f}, store issue {tr[:, 46].mean():.0f}, "
          f"other {tr[:, 47].mean():.0f}")


if __name__ == "__main__":
    main()
