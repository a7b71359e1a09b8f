"""Generate tests/golden/im2col_golden.json by running the REFERENCE's
GEMM-based path (im2col.py: build_patch_matrix, gemm_conv).

TEST INFRASTRUCTURE ONLY; run in the build container (the reference is
read-only at /root/reference, absent on the GPU box):

    python -m oracle.gen_golden_im2col

Per case: the seeded input (reference tensor_fill_random(shape, seed)),
filter (filter_fill_random(params, seed + 1)) and bias
(default_rng(seed + 2).uniform(-1, 1, K) as float32); recorded are SHA-256
digests of the reference patch matrix and of its gemm_conv output (float32,
little-endian).  They pin oracle/im2col.py (CPU) and the CUDA im2col +
GEMM-view path (tests/test_gpu_im2col.py) bit for bit.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from .gen_golden import OUT_DIR, REF_SRC, REF_TESTS, params_dict, sha

CASES = [
    # name, make_params kwargs, (n, h, w), seed
    ("3x3_p1", dict(r=3, s=3, pt=1, pl=1, c=8, k=16), (2, 6, 5), 11),
    ("strided_dilated_asym", dict(r=3, s=2, sy=2, sx=1, dy=2, dx=1, pt=2, pl=1, pb=0, pr=1, c=16, k=8), (1, 9, 7), 12),
    ("pointwise_view", dict(c=16, k=24), (2, 3, 4), 13),
    ("stem_like_7x7s2", dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=8), (1, 12, 10), 14),
    ("1x1_s2", dict(sy=2, sx=2, c=32, k=16), (2, 6, 6), 15),
]


def main() -> None:
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    import convbench as cb  # the reference
    from conftest import make_params  # reference test helper

    out = {"generator": "oracle/gen_golden_im2col.py", "reference": REF_SRC, "cases": []}
    for name, kw, (n, h, w), seed in CASES:
        p = make_params(**kw)
        shape = cb.Shape4(n, h, w, p.in_channels)
        inp = cb.tensor_fill_random(shape, seed)
        filt = cb.filter_fill_random(p, seed + 1)
        bias = np.random.default_rng(seed + 2).uniform(-1.0, 1.0, p.out_channels).astype(np.float32)
        tile = cb.TileConfig()
        pm = cb.build_patch_matrix(inp, p)
        mat = np.asarray(pm.matrix.base).reshape(pm.rows, pm.cols)
        pf = cb.pack_filter(filt, bias, p, tile)
        y = cb.gemm_conv(inp, pf, p, tile)
        out["cases"].append({
            "name": name, "params": params_dict(p), "shape": [n, h, w, p.in_channels], "seed": seed,
            "rows": int(pm.rows), "cols": int(pm.cols), "is_view": bool(pm.is_view),
            "patch_sha": sha(mat.astype("<f4")), "gemm_conv_sha": sha(np.asarray(y.data).astype("<f4")),
        })
    path = os.path.join(OUT_DIR, "im2col_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: {len(out['cases'])} cases")


if __name__ == "__main__":
    main()
