"""Clock-calibrated timeline of the window kernel (debug build with ICV_TRACE):
    ICV_LIB=.../libicv_trace.so python tools/trace_win.py cfg2
Warms the GPU up (clocks ramp) before the traced launch; prints per CTA the
phase times in SM cycles (clock64 / globaltimer ratio gives the clock)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200 import workloads as wl  # noqa: E402

# plan knobs for the run: ICV_KNOBS="win_mt=1,win_debug=1"
for _kv in filter(None, os.environ.get("ICV_KNOBS", "").split(",")):
    L.set_tuning(_kv.split("=")[0], int(_kv.split("=")[1]))

# ResNet-50 layers by name (not BASELINE configs): trace_win.py r50:s1b1_3x3
for _name, _shape, _params in wl.resnet50_layers(256):
    wl.CONFIGS["r50:" + _name] = wl.ConvWorkload("r50_" + _name, "bf16", _shape, _params)


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(300):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    flush_l2()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    tr = buf[:148].astype(np.int64)
    ok = tr[:, 61] > 0
    ghz = np.median((tr[ok, 60] - tr[ok, 62]) / (tr[ok, 61] - tr[ok, 0]))
    t0 = tr[ok, 0].min()
    rel = np.where(tr > 0, (tr - t0) * ghz, -1).astype(np.int64)   # cycles after the first entry
    print(f"{name}: clock {ghz:.3f} GHz; kernel span {(tr[ok, 61].max() - t0) / 1e3:.2f} us = {rel[ok, 61].max()} cycles")
    print(f"entry spread {rel[ok, 0].max()} cyc; setup median {np.median(rel[ok, 1] - rel[ok, 0]):.0f} cyc")
    for cta in (0, 2, 72, 146):
        r = rel[cta]
        units = [i for i in range(8) if r[2 + i] >= 0]
        row = " | ".join(f"u{i}: prod {r[26 + i]}-{r[40 + i]} mma_end {r[2 + i]} epi {r[10 + i]}-{r[18 + i]}"
                         for i in units)
        print(f"cta {cta:3d} entry {r[0]} setup {r[1]} end {r[61]} :: {row}")
    lead = tr[:, 34] > 0
    print(f"MMA warp (leaders): loop {tr[lead, 34].mean():.0f} cyc, waiting on full {tr[lead, 35].mean():.0f}, "
          f"on tmem-empty {tr[lead, 36].mean():.0f}")
    d = rel[:, 3] - rel[:, 2]
    print(f"median unit-1 mainloop {np.median(d[(d > 0) & lead]):.0f} cyc; "
          f"median epilogue {np.median((rel[:, 18] - rel[:, 10])[rel[:, 10] >= 0]):.0f} cyc")


if __name__ == "__main__" and not (len(sys.argv) > 2 and sys.argv[2] == "windows"):
    main()


def windows(name="cfg2"):
    """Per (unit, channel block) of CTA 0/2: window load issue -> stage full ->
    last MMA of the block issued (cycles after entry)."""
    main_args = sys.argv
    from paper_1907_02129_b200.workloads import CONFIGS

    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    for _ in range(300):
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    fn(None, 1)
    if not os.environ.get("NOFLUSH"):
        flush_l2()
    icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((1024, 128), np.uint64)
    fn(buf.ctypes.data, 0)
    tr = buf[:148].astype(np.int64)
    ok = tr[:, 61] > 0
    ghz = np.median((tr[ok, 60] - tr[ok, 62]) / (tr[ok, 61] - tr[ok, 0]))
    print(f"clock64 rate {ghz:.3f} GHz (undercounts: the counter stalls while every warp of the SM sleeps), "
          f"span {(tr[ok, 61].max() - tr[ok, 0].min()) / 1e3:.2f} us; times below in ns after CTA entry")
    ghz = 1.0
    for cta in (0, 2, 72):
        r = tr[cta]
        t0 = r[0]
        cells = []
        for k in range(8):
            if r[64 + k] == 0:
                continue
            iss, full, done = ((r[64 + k] - t0) * ghz, (r[72 + k] - t0) * ghz, (r[80 + k] - t0) * ghz)
            cells.append(f"u{k // 2}c{k % 2}: issue {iss:.0f} full {full:.0f} (+{full - iss:.0f}) mma_issued {done:.0f}")
        print(f"cta {cta}: " + " | ".join(cells))
        taps = [f"t{k}: +{r[96 + k] - t0} -> +{r[108 + k] - t0}" for k in range(12) if r[96 + k] or r[108 + k]]
        if taps:
            print(f"   unit 1, stage 0, per tap (filter block seen -> MMAs + commits issued, ns): " + ", ".join(taps))


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "windows":
    windows(sys.argv[1])
