"""Parity of the window kernel's stride-2 mode (phase planes; csrc/igemm_win.cu)
with the oracle.  The mode is opt-in (measured slower than the gather kernel
on B200 today); these tests force it with ICV_WIN=1.

A stride-2 layer is read as up to four phase planes of the input (rows of
parity py, columns of parity px), each a sliding-window operand on the output
grid; the cases cover which planes a kernel touches (3x3 pad 1: four; 2x2 pad
0: four with one tap each; dilation 2: one), asymmetric and odd padding,
odd image sizes, channel counts that are not a multiple of the 128-byte
block, output-channel tails, single CTA / CTA pairs, and uint8 with a zero
row holding the input zero point (TMA zero fill + the packed per-tap
correction) or all zeros (zero fill is exact) -- bit-exact against the
quantized oracle, including the BASELINE cfg4 geometry."""

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from helpers import assert_bf16_close
from oracle import conv as oconv
from oracle import quant as oq
from paper_1907_02129_b200 import _lib as L
from paper_1907_02129_b200.workloads import CFG4

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True)
def force_window(tune):
    tune(win=1)


S2_GEOMS = [
    dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=3, h=28, w=28, mr=128),                # ResNet-50 s2b1 3x3 shape
    dict(r=3, s=3, pt=1, pl=1, c=64, k=64, n=2, h=15, w=13, mr=4),                   # odd sizes, BN 64
    dict(r=3, s=3, dy=2, dx=2, pt=2, pl=2, c=256, k=256, n=2, h=20, w=18, mr=128),     # dilation 2: one plane
    dict(r=3, s=3, pt=0, pl=1, pb=1, pr=0, c=72, k=200, n=2, h=15, w=14, mr=3),       # asymmetric pads, C % 64, K tail
    dict(r=5, s=5, pt=2, pl=2, c=128, k=96, n=2, h=17, w=21, mr=128, gather=True),    # 5x5 (window does not fit)
    dict(r=2, s=2, c=32, k=40, n=3, h=12, w=12, mr=2),                                # 2x2 pad 0: one tap per plane
    dict(r=3, s=1, pt=1, pl=0, c=16, k=16, n=4, h=9, w=10, mr=5),                     # 3x1, column parity 0 only
]


def _params(g):
    g = dict(g)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    g.pop("mr", None)
    g.pop("gather", None)
    return make_params(sy=2, sx=2, **g), icv.Shape4(n, h, wd, g["c"])


def _bf16_case(g):
    p, shape = _params(g)
    rng = np.random.default_rng(23)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=g.get("mr", 128))
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile)
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), zero.float().cpu().numpy(), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    return p, shape, x, pf, ib, tile, ref


@pytest.mark.parametrize("geom", S2_GEOMS)
def test_stride2_window_matches_oracle(geom):
    p, shape, x, pf, ib, tile, ref = _bf16_case(geom)
    is_win = L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_win<bf16>"
    assert is_win != bool(geom.get("gather")), "case must exercise the window kernel (or, marked, must not)"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert_bf16_close(y, ref)


@pytest.mark.parametrize("cs,mt", [(1, 1), (1, 2), (2, 1), (2, 2)])
@pytest.mark.parametrize("geom", [S2_GEOMS[0], S2_GEOMS[3], S2_GEOMS[4]])
def test_stride2_window_variants(geom, cs, mt, tune):
    tune(win_cs=cs)
    tune(win_mt=mt)
    p, shape, x, pf, ib, tile, ref = _bf16_case(geom)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert_bf16_close(y, ref)


def test_stride2_window_equals_tap_gather():
    p, shape, x, pf, ib, tile, ref = _bf16_case(S2_GEOMS[0])
    y_win = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    ib.canonical = False
    y_gather = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    assert_bf16_close(y_win, y_gather)


def _u8_run(p, shape, zx, zw, zero_fill, seed=5):
    rng = np.random.default_rng(seed)
    xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
    wh = rng.integers(0, 256, p.out_channels * p.kernel_elems * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
    qp = icv.QuantParams(zx, 0.02, zw, 0.005, 128, 0.1)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=zero_fill)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oq.indirect_conv_u8(xh, zero.cpu().numpy(), ib.offsets_host(), p, wh, bias, shape.n, o.h, o.w,
                              zx, 0.02, zw, 0.005, 128, 0.1)
    return y, ref


def test_cfg4_window_selectable(tune):
    """uint8 takes the window kernel only when forced (ICV_WIN=1 here; the
    gather kernel is faster on cfg4 today)."""
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8) == "icv_igemm_win<u8>"
    tune(win=-1)
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8) == "icv_igemm_smem<u8,im2col>"
    tune(im2col_a=0)
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8) == "icv_igemm_smem<u8>"


@pytest.mark.parametrize("geom,zx,zw", [
    (dict(r=3, s=3, pt=1, pl=1, c=256, k=256, n=3, h=28, w=28), 128, 127),   # cfg4 geometry (BN 256, one accumulator)
    (dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=2, h=13, w=15), 3, 250),
    (dict(r=3, s=3, pt=0, pl=1, pb=1, pr=0, c=64, k=72, n=2, h=12, w=11), 200, 1),
    (dict(r=5, s=5, pt=2, pl=2, c=32, k=64, n=2, h=16, w=16), 255, 0),
])
@pytest.mark.parametrize("cs", [1, 2])
@pytest.mark.parametrize("cls", ["1", "0"])
def test_stride2_window_u8_zero_point_row(geom, zx, zw, cs, cls, tune):
    """Zero row = input zero point (the reference's quantized padding): TMA
    zero fill + padding correction (per border class, or per padded tap with
    ICV_WIN_U8_CLS=0) must give the oracle's bytes exactly."""
    tune(win_cs=cs)
    tune(win_u8_cls=int(cls))
    p, shape = _params(geom)
    y, ref = _u8_run(p, shape, zx, zw, zero_fill=zx)
    assert np.array_equal(y, ref), int((y != ref).sum())


def test_stride2_window_u8_zeros_row_nonzero_zp():
    """A zero row of zeros with zx != 0: padding really contributes
    (0 - zx)(w - zw); zero fill is then exact without correction."""
    p, shape = _params(dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=2, h=14, w=14))
    y, ref = _u8_run(p, shape, 128, 127, zero_fill=0)
    assert np.array_equal(y, ref), int((y != ref).sum())


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=128, k=256, h=14, w=14),                      # 9 border classes
    dict(r=3, s=3, pt=2, pl=2, dy=2, dx=2, c=128, k=256, h=13, w=12),          # 25 classes > RS: per-tap
    dict(r=3, s=3, pt=1, pl=0, pb=1, pr=2, c=64, k=128, h=11, w=10),           # asymmetric pads
    dict(r=3, s=3, pt=1, pl=1, c=64, k=64, h=3, w=2),                          # tiny: rows both top and bottom
])
@pytest.mark.parametrize("cls", ["1", "0"])
def test_stride1_window_u8_zero_point_row_pairs(geom, cls, tune):
    """Stride-1 uint8 with a zero-point zero row now also takes TMA windows
    (and CTA pairs) through the padding correction."""
    tune(win_cs=2)
    tune(win_u8_cls=int(cls))
    g = dict(geom)
    h, wd = g.pop("h"), g.pop("w")
    p = make_params(**g)
    y, ref = _u8_run(p, icv.Shape4(3, h, wd, g["c"]), 128, 127, zero_fill=128)
    assert np.array_equal(y, ref), int((y != ref).sum())


@pytest.mark.parametrize("geom,zx,zw", [
    (dict(r=3, s=3, pt=1, pl=1, c=256, k=256, n=3, h=28, w=28), 128, 127),   # cfg4 geometry
    (dict(r=3, s=3, pt=1, pl=0, pb=0, pr=1, c=64, k=512, n=2, h=9, w=11), 7, 200),
])
def test_u8_gather_kernel_block_n_256(geom, zx, zw, tune):
    """Opt-in BLOCK_N 256 of the uint8 gather kernel (two 256-column
    accumulator stages; the row sums come from the kernel's row-sum warps
    through shared memory instead of TMEM): bit-exact."""
    tune(win=0)
    tune(u8_bn=256)
    p, shape = _params(geom)
    y, ref = _u8_run(p, shape, zx, zw, zero_fill=zx)
    assert np.array_equal(y, ref), int((y != ref).sum())
