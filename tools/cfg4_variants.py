"""cfg4 timing under window-kernel plan knobs (A/B helper; icv_set_tuning)."""
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
W = {"win": 1}
runs = [("default dispatch", {}, False),
        ("window u8 (class corrections)", W, False),
        ("window u8 per-tap corrections", {**W, "win_u8_cls": 0}, False),
        ("window u8 BN128", {**W, "win_u8_bn": 128}, False),
        ("window u8 BN128 MT1", {**W, "win_u8_bn": 128, "win_mt": 1}, False),
        ("window u8 CS1", {**W, "win_cs": 1}, False),
        ("window u8 zeros-row flags (no corr; timing only)", W, True),
        ("gather kernel", {"win": 0}, False)]
for label, knobs, zeros in runs:
    zf, zz = ib.zero_fill_byte, ib.zero_is_zero
    if zeros:
        ib.zero_fill_byte, ib.zero_is_zero = None, True
    with icv._lib.tuning(**knobs):
        t = bench.time_steps(lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y), 20, 3, flush)
    ib.zero_fill_byte, ib.zero_is_zero = zf, zz
    print(f"{name} {label:45s} {statistics.median(t) * 1e3:8.2f} us")
