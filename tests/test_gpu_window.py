"""Parity of the stride-1 window kernel (csrc/igemm_win.cu) with the oracle.

The window kernel consumes a canonical indirection buffer of a stride-1
layer as one sliding window of padded input rows per tile; these cases cover
the geometry it has to get right: asymmetric padding (Zc = max(PL, PR)
shared zero columns), dilation, kernel sizes other than 3x3, channel counts
that are not a multiple of the 64-element block, output-channel tails at
BLOCK_N 64 / 128 / 256, odd M-tile counts (the second tile of a unit is a
dummy), a nonzero bf16 zero row (cp.async window gathers instead of TMA
zero-fill) and stride-1 uint8 (zero point fill, bit-exact)."""

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from helpers import assert_bf16_close
from oracle import conv as oconv
from oracle import quant as oq
from paper_1907_02129_b200 import _lib as L
from paper_1907_02129_b200.workloads import CFG2, CFG3B

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(autouse=True)
def force_window(tune):
    """ICV_WIN=1: the window kernel takes every stride-1 layer it fits, even
    small test images whose padded tiles are mostly discarded columns."""
    tune(win=1)

WIN_GEOMS = [
    dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=3, h=28, w=28, mr=128),            # cfg2 shape, 3 images
    dict(r=3, s=3, pt=1, pl=1, c=64, k=64, n=2, h=9, w=11, mr=4),                 # BN 64, tiny images
    dict(r=3, s=3, dy=2, dx=2, pt=2, pl=2, c=256, k=256, n=1, h=20, w=18, mr=128),  # dilation 2, BN 256
    dict(r=3, s=3, pt=1, pl=0, pb=0, pr=2, c=72, k=200, n=2, h=15, w=13, mr=3),   # asymmetric pads, C%64, K tail
    dict(r=5, s=3, dy=1, dx=3, pt=2, pl=3, pb=2, pr=3, c=48, k=96, n=2, h=12, w=20, mr=128),
    dict(r=1, s=1, c=64, k=128, n=2, h=16, w=16, mr=128),                         # pointwise
    dict(r=3, s=3, pt=1, pl=1, c=8, k=16, n=5, h=10, w=12, mr=7),                 # C = 8 (one 16-byte chunk)
    dict(r=2, s=2, pt=0, pl=0, pb=1, pr=1, c=32, k=40, n=3, h=11, w=11, mr=2),    # even kernel, bottom/right pad
]


def _bf16_case(g, zero_fill=0.0, index_dtype=torch.int64):
    g = dict(g)
    n, h, wd, mr = g.pop("n"), g.pop("h"), g.pop("w"), g.pop("mr")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(11)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=mr)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV, fill=zero_fill)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, index_dtype=index_dtype)
    return p, shape, xh, wh, bias, x, pf, zero, ib, tile, out_shape


def _oracle(p, shape, xh, wh, bias, zero, ib, o):
    return oconv.indirect_conv_f32(oconv.bf16_round(xh), zero.float().cpu().numpy(), ib.offsets_host(), p,
                                   oconv.bf16_round(wh), bias, shape.n, o.h, o.w)


def test_window_kernel_selected_for_stride1_baseline_configs():
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16) == "icv_igemm_win<bf16>"
    assert L.kernel_name(CFG3B.params, CFG3B.in_shape, torch.bfloat16) == "icv_igemm_win<bf16>"


@pytest.mark.parametrize("geom", WIN_GEOMS)
def test_window_kernel_matches_oracle(geom):
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _bf16_case(geom)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_win<bf16>", "case must exercise the window kernel"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert_bf16_close(y, _oracle(p, shape, xh, wh, bias, zero, ib, o))


@pytest.mark.parametrize("cs,mt", [(1, 1), (1, 2), (2, 1), (2, 2)])
@pytest.mark.parametrize("geom", [WIN_GEOMS[0], WIN_GEOMS[2], WIN_GEOMS[3], WIN_GEOMS[4]])
def test_window_kernel_variants(geom, cs, mt, tune):
    """Single CTA / CTA pair (cta_group::2, M = 256, filter rows split) x one /
    two M tiles per unit; odd image counts leave the pair's peer a dummy."""
    tune(win_cs=cs)
    tune(win_mt=mt)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _bf16_case(geom)
    assert ib.zero_is_zero
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert_bf16_close(y, _oracle(p, shape, xh, wh, bias, zero, ib, o))


@pytest.mark.parametrize("geom", [WIN_GEOMS[0], WIN_GEOMS[3], WIN_GEOMS[6]])
def test_window_kernel_nonzero_zero_row(geom):
    """Padding taps read the bound zero row (indirect.py:291): with a nonzero
    row the windows are gathered with cp.async from it (no TMA zero fill)."""
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _bf16_case(geom, zero_fill=0.75)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert_bf16_close(y, _oracle(p, shape, xh, wh, bias, zero, ib, o))


def test_window_kernel_equals_tap_gather():
    """Same sums as the tap-by-tap gather kernel (canonical flag cleared)."""
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _bf16_case(WIN_GEOMS[0])
    y_win = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    ib.canonical = False
    y_gather = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    assert_bf16_close(y_win, y_gather)


def test_window_kernel_batch_prefix():
    """batch < bound images: only the first `batch` images are convolved."""
    p, shape, xh, wh, bias, x, pf, zero, ib3, tile, o = _bf16_case(WIN_GEOMS[0])
    ib = icv.init_indirection_buffer(x, zero, p, o, tile, batch=2)
    y = icv.indirect_conv(x, pf, ib, p, tile, batch=2).numpy().reshape(-1, p.out_channels)
    ref = _oracle(p, shape, xh, wh, bias, zero, ib3, o).reshape(3, -1, p.out_channels)[:2].reshape(-1, p.out_channels)
    assert_bf16_close(y, ref)


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=64, k=64, n=3, h=14, w=14, zx=128, zw=127),
    dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=2, h=12, w=12, zx=3, zw=250),
    dict(r=3, s=3, dy=2, dx=2, pt=2, pl=2, c=48, k=40, n=2, h=11, w=12, zx=0, zw=9),
])
def test_window_kernel_u8_bit_exact(geom):
    g = dict(geom)
    n, h, wd, zx, zw = (g.pop(k) for k in ("n", "h", "w", "zx", "zw"))
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    assert L.kernel_name(p, shape, torch.uint8) == "icv_igemm_win<u8>"
    rng = np.random.default_rng(5)
    xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
    wh = rng.integers(0, 256, p.out_channels * p.kernel_elems * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
    qp = icv.QuantParams(zx, 0.02, zw, 0.005, 128, 0.1)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=zx)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oq.indirect_conv_u8(xh, zero.cpu().numpy(), ib.offsets_host(), p, wh, bias, n, o.h, o.w,
                              zx, 0.02, zw, 0.005, 128, 0.1)
    assert np.array_equal(y, ref), int((y != ref).sum())


@pytest.mark.parametrize("geom", [dict(r=3, s=3, pt=1, pl=1, c=64, k=64, n=32, h=56, w=56, mr=128),
                                  dict(r=3, s=3, pt=1, pl=1, c=256, k=256, n=64, h=14, w=14, mr=128)])
def test_window_kernel_full_size_equals_gather(geom, tune):
    """ResNet-50 stride-1 3x3 shapes at full size (many units per CTA: the
    filter ring and the resident-filter plans wrap many times) agree with the
    IB-gather kernel."""
    tune(win=-1)
    tune(im2col_a=0)   # (the auto plan gives the 256-channel 14x14 shape to the im2col TMA kernel)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _bf16_case(geom)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_win<bf16>"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    yg = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert_bf16_close(y, yg)
