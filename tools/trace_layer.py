"""Per-CTA timeline of the tensor-core gather / dense kernel on one cfg5
layer (debug build with ICV_TRACE):
    ICV_LIB=.../libicv_trace.so python tools/trace_layer.py s1b1_1x1b"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200.stack import ResNet50Stack  # noqa: E402


def main():
    name = sys.argv[1]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    stack = ResNet50Stack(batch=batch, device=dev)
    layer = {l.name: l for l in stack.layers}[name]
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(3):
        stack.run_layer(layer)
    fn(None, 1)
    flush_l2()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    stack.run_layer(layer)
    e.record()
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    tr = buf[:148].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = np.where(tr > 0, tr - t0, -1)
    print(f"{name}: event {s.elapsed_time(e) * 1e3:.1f} us; kernel entry spread {(rel[:, 0].max()) / 1e3:.2f} us; "
          f"setup {np.median(rel[:, 1] - rel[:, 0]) / 1e3:.2f} us")
    for cta in (0, 1, 73, 147):
        r = rel[cta]
        tiles = [i for i in range(8) if r[2 + i] >= 0]
        row = " | ".join(f"t{i}: prod {r[26 + i] / 1e3:.2f}-{r[40 + i] / 1e3:.2f} "
                         f"mma_end {r[2 + i] / 1e3:.2f} epi {r[10 + i] / 1e3:.2f}-{r[18 + i] / 1e3:.2f}"
                         for i in tiles)
        print(f"cta {cta:3d} entry {r[0] / 1e3:.2f} setup {r[1] / 1e3:.2f} :: {row}")
    cyc = buf[:148, 34].astype(np.float64)
    wf = buf[:148, 35].astype(np.float64)
    wt = buf[:148, 36].astype(np.float64)
    ns = (tr[:, 2:10].max(axis=1) - tr[:, 1]).astype(np.float64)
    print(f"MMA warp: loop {cyc.mean():.0f} cycles (mean), waiting on full {wf.mean():.0f}, on tmem-empty {wt.mean():.0f}; "
          f"effective clock ~{np.median(cyc / np.maximum(ns, 1)):.2f} GHz")
    pl = buf[:148, 37].astype(np.float64)
    pw = buf[:148, 38].astype(np.float64)
    print(f"producer thread 0: loop {pl.mean():.0f} cycles, waiting on empty {pw.mean():.0f}")
    ew = buf[:148, 28].astype(np.float64)
    ek = buf[:148, 29].astype(np.float64)
    print(f"epilogue warp 0: waiting on tmem-full {ew.mean():.0f} cycles, working {ek.mean():.0f} cycles")
    for cta in (0, 1):
        r = tr[cta]
        print(f"cta {cta}: per stage of the traced tile (us after entry): free / issued / full")
        for s_ in range(16):
            if r[64 + s_] == 0 and r[80 + s_] == 0:
                break
            f = lambda v: f"{(v - r[0]) / 1e3:7.2f}" if v > 0 else "      -"   # noqa: E731
            print(f"   s{s_:2d}: {f(r[64 + s_])} {f(r[96 + s_])} {f(r[80 + s_])}")
    d = rel[:, 3] - rel[:, 2]
    print(f"median tile-1 mainloop (mma_end1 - mma_end0) {np.median(d[d > 0]) / 1e3:.2f} us; "
          f"median epilogue {np.median((rel[:, 18] - rel[:, 10])[rel[:, 10] >= 0]) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
