"""Per-tile timeline of the row-sliding kernel (build with -DICV_ROWS_TIMELINE):
us after CTA entry when the loader issued tile k, the converters finished it,
the MMA warp committed it and epilogue warp 0 released its accumulator."""
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
    t_all = buf[:148, 0][buf[:148, 0] > 0].min()
    for cta in (0, 1, 77):
        r = buf[cta].astype(np.int64)
        t0 = r[0]
        print(f"cta {cta}: entry {(t0 - t_all) / 1e3:.2f} us, setup done {(r[1] - t0) / 1e3:.2f}")
        print("   k   load   conv    mma    epi (us after entry)")
        for k in range(24):
            if r[8 + k] == 0:
                break
            f = lambda v: f"{(v - t0) / 1e3:6.2f}" if v else "   -  "
            print(f"  {k:2d} {f(r[8 + k])} {f(r[32 + k])} {f(r[56 + k])} {f(r[80 + k])}")


if __name__ == "__main__":
    main()
