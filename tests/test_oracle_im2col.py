"""oracle/im2col.py against the reference's own GEMM-based path
(tests/golden/im2col_golden.json, made by oracle/gen_golden_im2col.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import make_params
from oracle import im2col as oi
from oracle.gen_golden import sha

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "im2col_golden.json")))


def _case_inputs(case):
    p = make_params(**{k: v for k, v in _kw(case["params"]).items()})
    n, h, w, c = case["shape"]
    seed = case["seed"]
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, n * h * w * c).astype(np.float32)       # tensors.py:219-223
    wk = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, p.out_channels * p.kernel_h * p.kernel_w * c).astype(np.float32)
    bias = np.random.default_rng(seed + 2).uniform(-1.0, 1.0, p.out_channels).astype(np.float32)
    return p, (n, h, w), x, wk, bias


def _kw(pd):
    return dict(r=pd["kernel_h"], s=pd["kernel_w"], sy=pd["stride_h"], sx=pd["stride_w"], dy=pd["dilation_h"],
                dx=pd["dilation_w"], pt=pd["pad_top"], pl=pd["pad_left"], pb=pd["pad_bottom"], pr=pd["pad_right"],
                c=pd["in_channels"], k=pd["out_channels"])


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_oracle_im2col_matches_reference(case):
    p, (n, h, w), x, wk, bias = _case_inputs(case)
    mat = oi.patch_matrix(x, p, n, h, w)
    assert mat.shape == (case["rows"], case["cols"])
    assert sha(mat.astype("<f4")) == case["patch_sha"]
    assert sha(oi.gemm_conv_f32(mat, wk, bias).astype("<f4")) == case["gemm_conv_sha"]
