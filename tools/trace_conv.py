"""Per-CTA timeline of the tcgen05 kernel (debug build with ICV_TRACE):
    ICV_LIB=.../libicv_trace.so python tools/trace_conv.py cfg2"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402

# plan knobs for the run: ICV_KNOBS="cluster=2,u8_bn=256"
for _kv in filter(None, os.environ.get("ICV_KNOBS", "").split(",")):
    L.set_tuning(_kv.split("=")[0], int(_kv.split("=")[1]))


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(3):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    flush_l2()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    e.record()
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    tr = buf[:148].astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = np.where(tr > 0, tr - t0, -1)
    print(f"{name}: event {s.elapsed_time(e) * 1e3:.1f} us; kernel entry spread {(rel[:, 0].max()) / 1e3:.2f} us; "
          f"setup {np.median(rel[:, 1] - rel[:, 0]) / 1e3:.2f} us")
    last_end = rel[:, 18:26].max()
    print(f"last epilogue release at {last_end / 1e3:.2f} us after first CTA entry")
    for cta in (0, 1, 73, 147):
        r = rel[cta]
        tiles = [i for i in range(8) if r[2 + i] >= 0]
        row = " | ".join(f"t{i}: prod {r[26 + i] / 1e3:.2f}-{r[40 + i] / 1e3:.2f} slice {r[48 + i] / 1e3:.2f} "
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
    d = rel[:, 3] - rel[:, 2]
    print(f"median tile-1 mainloop (mma_end1 - mma_end0) {np.median(d[d > 0]) / 1e3:.2f} us; "
          f"median epilogue {np.median((rel[:, 18] - rel[:, 10])[rel[:, 10] >= 0]) / 1e3:.2f} us")


if __name__ == "__main__" and not (len(sys.argv) > 2 and sys.argv[2] == "stages"):
    main()


def stages(name="cfg2"):
    """Per-stage timeline of tile 1 (CTA 0..3): stage free -> issued -> full."""
    from paper_1907_02129_b200.workloads import CONFIGS

    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(3):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    flush_l2()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    for cta in range(4):
        r = buf[cta].astype(np.int64)
        t0 = r[0]
        print(f"cta {cta}: (us after entry) free / issued / full per stage")
        for s_ in range(12):
            if r[64 + s_] == 0:
                break
            print(f"   s{s_:2d}: {(r[64 + s_] - t0) / 1e3:7.2f} {(r[96 + s_] - t0) / 1e3:7.2f} {(r[80 + s_] - t0) / 1e3:7.2f}")


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "stages":
    stages(sys.argv[1])
