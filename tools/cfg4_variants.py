"""cfg4 timing under window-kernel knobs (A/B helper)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200.workloads import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
dev = torch.device("cuda", 0)
w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
flush = bench.make_l2_flush(dev)
W = {"ICV_WIN": "1"}
runs = [("default dispatch", {}, False),
        ("window u8 (class corrections)", W, False),
        ("window u8 per-tap corrections", {**W, "ICV_WIN_U8_CLS": "0"}, False),
        ("window u8 BN128", {**W, "ICV_WIN_U8_BN": "128"}, False),
        ("window u8 BN128 MT1", {**W, "ICV_WIN_U8_BN": "128", "ICV_WIN_MT": "1"}, False),
        ("window u8 CS1", {**W, "ICV_WIN_CS": "1"}, False),
        ("window u8 zeros-row flags (no corr; timing only)", W, True),
        ("gather kernel", {"ICV_WIN": "0"}, False)]
for label, env, zeros in runs:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    zf, zz = ib.zero_fill_byte, ib.zero_is_zero
    if zeros:
        ib.zero_fill_byte, ib.zero_is_zero = None, True
    t = bench.time_steps(lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y), 20, 3, flush)
    ib.zero_fill_byte, ib.zero_is_zero = zf, zz
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    print(f"{name} {label:45s} {statistics.median(t) * 1e3:8.2f} us")
