"""cfg4 timing of the IB-gather kernel under its plan knobs (A/B helper; icv_set_tuning)."""
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
runs = [("default", {}), ("BN256", {"u8_bn": 256}), ("pair", {"cluster": 2}), ("pair BN256", {"cluster": 2, "u8_bn": 256})]
ref = None
for label, knobs in runs:
    with icv._lib.tuning(**knobs):
        t = bench.time_steps(lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y), 20, 3, flush)
        torch.cuda.synchronize()
        out = y.data.clone()
    if ref is None:
        ref = out
    same = bool(torch.equal(ref, out))
    print(f"{name} {label:20s} {statistics.median(t) * 1e3:8.2f} us  equal_to_default={same}")
