"""GEMM-based baseline on the device (paper_1907_02129_b200/im2col.py, csrc/im2col.cu)
against the reference's build_patch_matrix / gemm_conv (golden digests from
oracle/gen_golden_im2col.py) and against indirect_conv on the same inputs."""

import json
import os

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from helpers import assert_bf16_close
from oracle import im2col as oi
from oracle.gen_golden import sha
from test_oracle_im2col import _kw

pytestmark = pytest.mark.gpu
DEV = "cuda"
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "im2col_golden.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_gpu_patch_matrix_and_gemm_conv_bitexact_vs_reference(case):
    p = make_params(**_kw(case["params"]))
    n, h, w, c = case["shape"]
    seed = case["seed"]
    x = icv.tensor_fill_random(icv.Shape4(n, h, w, c), seed, device=DEV)
    pm = icv.build_patch_matrix(x, p)
    assert (pm.rows, pm.cols, pm.is_view) == (case["rows"], case["cols"], case["is_view"])
    assert sha(pm.matrix.cpu().numpy().astype("<f4")) == case["patch_sha"]
    filt = icv.filter_fill_random(p, seed + 1, device=DEV)
    bias = np.random.default_rng(seed + 2).uniform(-1.0, 1.0, p.out_channels).astype(np.float32)
    tile = icv.TileConfig()
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile)
    y = icv.gemm_conv(x, pf, p, tile)
    assert sha(y.numpy().astype("<f4")) == case["gemm_conv_sha"]


def test_gpu_patch_matrix_refill_and_zero_row():
    p = make_params(r=3, s=3, pt=1, pl=1, c=16, k=8)
    x = icv.tensor_fill_random(icv.Shape4(2, 5, 7, 16), 3, device=DEV, dtype=torch.bfloat16)
    pm = icv.build_patch_matrix(x, p)
    x2 = icv.tensor_fill_random(icv.Shape4(2, 5, 7, 16), 4, device=DEV, dtype=torch.bfloat16)
    same = icv.build_patch_matrix(x2, p, out=pm)
    assert same is pm
    ref = oi.patch_matrix(x2.data.float().cpu().numpy(), p, 2, 5, 7)
    assert np.array_equal(pm.matrix.float().cpu().numpy(), ref)
    z = torch.full((16,), 7, dtype=torch.uint8, device=DEV)
    xu = icv.NhwcTensor(icv.Shape4(1, 4, 4, 16), torch.randint(0, 256, (256,), dtype=torch.uint8, device=DEV))
    pmu = icv.build_patch_matrix(xu, p, zero_row=z)
    refu = oi.patch_matrix(xu.data.cpu().numpy(), p, 1, 4, 4, pad=np.full(16, 7, np.uint8))
    assert np.array_equal(pmu.matrix.cpu().numpy(), refu)
    with pytest.raises(ValueError):
        icv.build_patch_matrix(x2, make_params(r=3, s=3, c=16, k=8), out=pm)


def test_gpu_gemm_conv_bf16_matches_indirect():
    """cfg2-shaped (fewer images): the two variants compute the same sums."""
    p = make_params(r=3, s=3, pt=1, pl=1, c=128, k=128)
    shape = icv.Shape4(4, 28, 28, 128)
    rng = np.random.default_rng(0)
    x = icv.NhwcTensor(shape, torch.from_numpy(rng.standard_normal(shape.numel, dtype=np.float32)).to(DEV)
                       .to(torch.bfloat16))
    wt = torch.from_numpy(rng.standard_normal(128 * 9 * 128, dtype=np.float32) * np.float32(np.sqrt(2 / 1152)))
    filt = icv.FilterTensor(128, 3, 3, 128, wt.to(DEV))
    tile = icv.TileConfig(mr=128)
    pf = icv.pack_filter(filt, None, p, tile, compute_dtype=torch.bfloat16)
    y_gemm = icv.gemm_conv(x, pf, p, tile).numpy()
    zero = icv.make_zero_row(128, dtype=torch.bfloat16, device=DEV)
    ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), tile)
    y_ind = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    assert_bf16_close(y_gemm, y_ind)


@pytest.mark.parametrize("geom", [dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=64, k=64, h=14, w=14),
                                  dict(r=3, s=3, pt=1, pl=1, c=32, k=48, h=9, w=11)])
def test_gpu_gemm_conv_u8_equals_indirect(geom):
    """uint8: padding taps take the zero point in the patch matrix, so the
    GEMM baseline equals the indirect convolution byte for byte."""
    g = dict(geom)
    h, w = g.pop("h"), g.pop("w")
    p = make_params(**g)
    shape = icv.Shape4(2, h, w, p.in_channels)
    rng = np.random.default_rng(9)
    xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
    wh = rng.integers(0, 256, p.out_channels * p.kernel_elems * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
    qp = icv.QuantParams(128, 0.02, 127, 0.005, 128, 0.1)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=128)
    ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), tile)
    y_ind = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    y_gemm = icv.gemm_conv(x, pf, p, tile).numpy()
    assert np.array_equal(y_gemm, y_ind)
