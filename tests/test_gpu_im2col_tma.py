"""Parity of the im2col-TMA A mode of the tensor-core kernel (csrc/igemm_tc.cu,
tma_a_mode 2) with the oracle and, bit for bit, with the IB-gather kernel.

Over a canonical indirection buffer with an all-zero zero row, the references
of an M tile are a function of the geometry (indirect.py:112-125), so the TMA
unit can generate them itself: one im2col tile load per (tap, channel block)
brings the 128 output pixels' input rows, zero-filled where the tap leaves
the image.  The accumulation order (tap-major, channel block, 32-byte K
steps) is the gather kernel's, so the two must agree byte for byte.  Cases:
stride 2 (both and one direction), strided 1x1 (the ResNet projections),
dilation, asymmetric padding, odd sizes, tiles that span several images,
K tails, single CTAs and CTA pairs, int32 and per-image buffers, and the
fallbacks (non-zero zero row, forged buffer, partial channel block)."""

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from helpers import assert_bf16_close
from oracle import conv as oconv
from paper_1907_02129_b200 import _lib as L

pytestmark = pytest.mark.gpu
DEV = "cuda"

GEOMS = [
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=128, k=128, n=3, h=28, w=28),              # ResNet-50 s2b1 3x3
    dict(r=1, s=1, sy=2, sx=2, c=256, k=512, n=2, h=14, w=14),                          # strided projection
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=64, k=64, n=2, h=9, w=11),                 # odd sizes, BN 64
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=512, k=512, n=7, h=14, w=14),              # 49-pixel images: tiles span images
    dict(r=5, s=3, sy=2, sx=2, pt=2, pl=1, pb=1, pr=2, c=64, k=40, n=2, h=17, w=21),    # 5x3, asymmetric pads, K tail
    dict(r=3, s=3, sy=2, sx=1, pt=1, pl=1, c=64, k=96, n=2, h=12, w=10),                # stride 2 in y only
    dict(r=3, s=3, sy=1, sx=3, dy=2, dx=1, pt=2, pl=0, pb=2, pr=2, c=128, k=64, n=2, h=11, w=13),   # stride 3, dilation
    dict(r=4, s=6, sy=2, sx=2, pt=1, pl=3, pb=2, pr=2, c=64, k=64, n=1, h=20, w=20),    # 24 taps (the kernels' limit)
    dict(r=2, s=2, sy=2, sx=2, c=64, k=64, n=3, h=8, w=8),                              # 2x2 pad 0
]


def _case(g, index_dtype=torch.int64, per_image=True):
    g = dict(g)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p, shape = make_params(**g), icv.Shape4(n, h, wd, g["c"])
    rng = np.random.default_rng(29)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile, index_dtype=index_dtype, per_image=per_image)
    return p, shape, xh, wh, bias, x, pf, zero, ib, tile, o


@pytest.mark.parametrize("cs", [1, 2])
@pytest.mark.parametrize("geom", GEOMS)
def test_im2col_tma_matches_oracle_and_gather(geom, cs, tune):
    tune(dense_cs=cs)
    tune(im2col_a=2)   # (wherever eligible: the auto plan takes it from four channel blocks up)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom)
    name = L.kernel_name(p, shape, torch.bfloat16)
    assert name == ("icv_igemm_smem<bf16,im2col,pair>" if cs == 2 else "icv_igemm_smem<bf16,im2col>"), name
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(p.in_channels, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    assert_bf16_close(y.reshape(-1, p.out_channels), ref.reshape(-1, p.out_channels))
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y.tobytes() == y_gather.tobytes()


def test_im2col_tma_int32_canonical_buffer(tune):
    tune(im2col_a=2)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(GEOMS[0], index_dtype=torch.int32, per_image=False)
    assert "im2col" in L.kernel_name(p, shape, torch.bfloat16, L.DEFAULT_FLAGS & ~L.ICV_IB_PER_IMAGE)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y.tobytes() == y_gather.tobytes()


def test_im2col_tma_auto_plan(tune):
    """Auto (im2col_a = 1): from four channel blocks up where the IB gather
    would run, and instead of the window kernel when the output rows are short."""
    def name(**g):
        n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
        return L.kernel_name(make_params(**g), icv.Shape4(n, h, wd, g["c"]), torch.bfloat16)
    assert name(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=128, k=128, n=2, h=28, w=28) == "icv_igemm_smem<bf16>"
    assert name(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=256, k=256, n=2, h=28, w=28) == "icv_igemm_smem<bf16,im2col,pair>"
    assert name(r=1, s=1, sy=2, sx=2, c=256, k=512, n=2, h=56, w=56) == "icv_igemm_smem<bf16,im2col,pair>"
    assert name(r=3, s=3, pt=1, pl=1, c=256, k=256, n=2, h=14, w=14) == "icv_igemm_smem<bf16,im2col,pair>"
    assert name(r=3, s=3, pt=1, pl=1, c=256, k=256, n=2, h=28, w=28) == "icv_igemm_win<bf16>"
    assert name(r=3, s=3, pt=1, pl=1, c=128, k=128, n=2, h=14, w=14) == "icv_igemm_win<bf16>"


def test_im2col_tma_instead_of_the_window_kernel(tune):
    """Knob im2col_a = 2 takes the im2col kernel where the window kernel would run (A/B)."""
    g = dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=3, h=28, w=28)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(g)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_win<bf16>"
    y_win = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    tune(im2col_a=2)
    assert "im2col" in L.kernel_name(p, shape, torch.bfloat16)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y.tobytes() == y_gather.tobytes()
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(p.in_channels, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    assert_bf16_close(y.reshape(-1, p.out_channels), ref.reshape(-1, p.out_channels))
    assert_bf16_close(y_win.reshape(-1, p.out_channels), ref.reshape(-1, p.out_channels))


def test_im2col_tma_fallbacks(tune):
    """The IB-gather kernel keeps: buffers that are not canonical, zero rows
    that are not all zeros, partial channel blocks, and im2col_a = 0."""
    tune(im2col_a=2)
    g = GEOMS[0]
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(g)
    flags = L.DEFAULT_FLAGS
    assert "im2col" in L.kernel_name(p, shape, torch.bfloat16, flags)
    assert L.kernel_name(p, shape, torch.bfloat16, flags & ~L.ICV_IB_CANONICAL) == "icv_igemm_smem<bf16>"
    assert L.kernel_name(p, shape, torch.bfloat16, flags & ~L.ICV_ZERO_ROW_ZEROS) == "icv_igemm_smem<bf16>"
    g72 = dict(g, c=72)
    p72, shape72 = make_params(**{k: v for k, v in g72.items() if k not in ("n", "h", "w")}), icv.Shape4(3, 28, 28, 72)
    assert L.kernel_name(p72, shape72, torch.bfloat16) == "icv_igemm_smem<bf16>"
    tune(im2col_a=0)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_smem<bf16>"
    # a non-zero zero row is followed (the reference reads it for padding taps)
    tune(im2col_a=2)
    zero1 = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    zero1.fill_(0.5)
    ib1 = icv.init_indirection_buffer(x, zero1, p, o, tile)
    y1 = icv.indirect_conv(x, pf, ib1, p, tile).numpy()
    ref1 = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.full(p.in_channels, 0.5, np.float32), ib1.offsets_host(), p,
                                   oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    assert_bf16_close(y1.reshape(-1, p.out_channels), ref1.reshape(-1, p.out_channels))


# ---------------------------------------------------------------- uint8
# Zero row = input zero point (the QNNPACK convention): TMA zero-fills the
# padded taps instead, and the epilogue adds, per border class of the pixel,
# what those taps would have contributed.  Bit-exact against the quantized
# oracle, which follows the buffer and the zero row.
U8_GEOMS = [
    (dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=256, k=256, n=3, h=28, w=28), 128, 127),      # cfg4 geometry: 2 x 2 classes
    (dict(r=3, s=3, pt=1, pl=1, c=128, k=128, n=2, h=9, w=11), 3, 200),                     # stride 1: 3 x 3 classes
    (dict(r=1, s=1, sy=2, sx=2, c=128, k=64, n=2, h=10, w=10), 7, 9),                       # strided 1x1: no padding
    (dict(r=3, s=5, sy=2, sx=1, dy=2, dx=1, pt=2, pl=1, pb=3, pr=3, c=128, k=40, n=2, h=13, w=9), 128, 1),   # asymmetric
    (dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=256, k=512, n=5, h=6, w=6), 255, 0),           # 3x3 outputs: every pixel a border pixel
]


def _u8_case(g, zx, zw, zero_fill):
    from oracle import quant as oq

    g = dict(g)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p, shape = make_params(**g), icv.Shape4(n, h, wd, g["c"])
    rng = np.random.default_rng(31)
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
    ref = oq.indirect_conv_u8(xh, zero.cpu().numpy(), ib.offsets_host(), p, wh, bias, shape.n, o.h, o.w,
                              zx, 0.02, zw, 0.005, 128, 0.1)
    return p, shape, x, pf, ib, tile, ref


@pytest.mark.parametrize("cs", [1, 2])
@pytest.mark.parametrize("geom,zx,zw", U8_GEOMS)
def test_im2col_tma_u8_bit_exact(geom, zx, zw, cs, tune):
    tune(dense_cs=cs)
    p, shape, x, pf, ib, tile, ref = _u8_case(geom, zx, zw, zx)
    name = L.kernel_name(p, shape, torch.uint8)
    assert name == ("icv_igemm_smem<u8,im2col,pair>" if cs == 2 else "icv_igemm_smem<u8,im2col>"), name
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert np.array_equal(y, ref), int((y != ref).sum())
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy().reshape(-1, p.out_channels)
    assert np.array_equal(y_gather, ref)


def test_im2col_tma_u8_other_zero_rows_keep_the_gather(tune):
    """A uint8 zero row that is neither all zeros nor the zero point is followed through the buffer."""
    g, zx, zw = U8_GEOMS[0]
    p, shape, x, pf, ib, tile, ref = _u8_case(g, zx, zw, 77)
    assert L.kernel_name(p, shape, torch.uint8, L.ICV_IB_CANONICAL | L.ICV_IB_PER_IMAGE) == "icv_igemm_smem<u8>"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    assert np.array_equal(y, ref), int((y != ref).sum())


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=256, k=256, n=64, h=14, w=14),                    # ResNet-50 s3 3x3 (instead of the window kernel)
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=512, k=512, n=64, h=14, w=14),        # s4b1 3x3 / 2
    dict(r=1, s=1, sy=2, sx=2, c=512, k=1024, n=32, h=28, w=28),                   # s3b1 projection
])
def test_im2col_tma_full_size_equals_gather(geom):
    """ResNet-50 shapes at a batch where every CTA pair runs several tiles (the
    stage ring wraps many times, odd tile counts leave a dummy tile): the
    automatic plan takes the im2col pair kernel and agrees with the IB-gather
    kernel byte for byte."""
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_smem<bf16,im2col,pair>"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y.tobytes() == y_gather.tobytes()


def test_im2col_tma_random_geometries():
    """Randomized sweep (tools/fuzz_im2col.py): 150 random geometries, bf16 and
    uint8, single CTAs and pairs, all equal to the IB-gather kernel."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_im2col

    ran, bad = fuzz_im2col.run(150, 7)
    assert bad == 0
    assert ran["bf16"] >= 150 and ran["u8"] >= 80
