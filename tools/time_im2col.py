"""Split of the GEMM-based baseline on a BASELINE config: patch-matrix build
(icv_im2col, HBM-bound) vs the GEMM over it, CUDA events, L2 flushed."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200.workloads import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
dev = torch.device("cuda", 0)
w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev)
flush = bench.make_l2_flush(dev)
pm = icv.build_patch_matrix(x, w.params)
icv.gemm_only(pm, pf, tile)
tb = statistics.median(bench.time_steps(lambda: icv.build_patch_matrix(x, w.params, out=pm), 20, 3, flush))
tg = statistics.median(bench.time_steps(lambda: icv.gemm_only(pm, pf, tile), 20, 3, flush))
mb = pm.allocated_bytes / 1e6
print(f"{name}: im2col {tb * 1e3:.2f} us ({mb:.1f} MB written, {mb / 1e3 / (tb * 1e-3):.0f} GB/s), "
      f"gemm {tg * 1e3:.2f} us ({w.flops / (tg * 1e-3) / 1e12:.0f} TFLOP/s)")
