"""SM clock during the bench's own timing loop (debug build with ICV_TRACE):
    ICV_LIB=.../libicv_trace.so python tools/clock_probe.py cfg2
Runs bench.time_steps' sequence (flush, event, conv, event) and reads, after
every step, the window kernel's clock64 / globaltimer stamps (slots 60-62, 0):
cycles per nanosecond over the kernel = the SM clock the step actually ran at."""
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

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    mode = sys.argv[2] if len(sys.argv) > 2 else "flush"
    dev = torch.device("cuda", 0)
    w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
    fn = L.lib().icv_debug_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush_l2 = bench.make_l2_flush(dev)
    buf = np.zeros((1024, 128), np.uint64)
    for step in range(12):
        if mode == "flush":
            flush_l2()
        elif mode == "busy":      # keep the tensor cores busy before the step
            a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
            for _ in range(20):
                a @ a
        fn(None, 1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        icv.indirect_conv(x, pf, ib, w.params, tile, out=y)
        e.record()
        torch.cuda.synchronize()
        fn(buf.ctypes.data, 0)
        tr = buf[:148].astype(np.int64)
        ok = tr[:, 61] > 0
        ghz = np.median((tr[ok, 60] - tr[ok, 62]) / (tr[ok, 61] - tr[ok, 0]))
        span_ns = tr[ok, 61].max() - tr[ok, 0].min()
        cyc = (tr[ok, 60] - tr[ok, 62]).max()
        print(f"{name} [{mode}] step {step:2d}: event {s.elapsed_time(e) * 1e3:6.2f} us  kernel span {span_ns / 1e3:6.2f} us  "
              f"{cyc} cycles  SM clock {ghz:.3f} GHz")


if __name__ == "__main__":
    main()
