"""Host-side cost of one indirect_conv call (Python API and bare C ABI),
measured without synchronizing: the GPU work is queued, not waited for."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    n = 200
    for _ in range(10):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    d, s = L.desc_of(w.params), L.shape_of(x.shape)
    args = (ctypes.byref(d), ctypes.byref(s), x.shape.n, L.TORCH_TO_ICV[x.dtype], L.ptr(x.data), L.ptr(ib.zero_row),
            L.ptr(ib.offsets), L.TORCH_TO_ICV[ib.offsets.dtype] | (L.ICV_IB_PER_IMAGE if ib.per_image else 0), ib.mr,
            L.ptr(pf.packed), None, L.ptr(y.data), L.stream_of(dev))
    fn = L.lib().icv_conv
    t2 = time.perf_counter()
    for _ in range(n):
        fn(*args)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: indirect_conv {1e6 * (t1 - t0) / n:.1f} us/call host, bare icv_conv {1e6 * (t3 - t2) / n:.1f} us/call")


if __name__ == "__main__":
    main()
