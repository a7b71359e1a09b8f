"""Dense-A mode of the tensor-core kernel: 1x1, stride-1, unpadded layers over
a canonical buffer load the A tile as TMA boxes of 128 consecutive pixel rows
(the buffer's entries are p -> p, reference indirect.py:112-125 with
R = S = 1).  Checked against the oracle and, bit for bit, against the
IB-gather kernel on the same inputs (same A bytes, same MMA order)."""

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from helpers import assert_bf16_close
from oracle import conv as oconv
from oracle import quant as oq
from paper_1907_02129_b200 import _lib as L

pytestmark = pytest.mark.gpu
DEV = "cuda"

DENSE_GEOMS = [
    dict(c=64, k=64, n=3, h=28, w=28),      # BN 64, 1 K block, P % 128 != 0
    dict(c=64, k=256, n=2, h=14, w=14),     # BN 256, 8 epilogue warps (K >= 4C)
    dict(c=256, k=64, n=2, h=14, w=14),     # 4 K blocks
    dict(c=72, k=40, n=1, h=9, w=7),        # partial channel block (TMA zero fill past C), K tail
    dict(c=8, k=16, n=2, h=5, w=3),         # one 16-byte chunk per row
    dict(c=512, k=1024, n=1, h=7, w=7),     # 4 N tiles, 8 K blocks
]


def _case(g, per_image, index_dtype, seed=3):
    g = dict(g)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(seed)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, 1, 1, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile, index_dtype=index_dtype, per_image=per_image)
    return p, shape, xh, wh, bias, x, pf, zero, ib, tile, o


@pytest.mark.parametrize("cs", [1, 2])
@pytest.mark.parametrize("per_image,index_dtype", [(True, torch.int64), (False, torch.int32)])
@pytest.mark.parametrize("geom", DENSE_GEOMS)
def test_dense_a_matches_oracle_and_gather(geom, per_image, index_dtype, cs, tune):
    """Single CTAs and CTA pairs (cta_group::2, M = 256, each CTA its own
    rows and half the filter block; odd M-tile counts leave a dummy)."""
    tune(dense_cs=cs)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom, per_image, index_dtype)
    assert L.kernel_name(p, shape, torch.bfloat16) == ("icv_igemm_smem<bf16,dense,pair>" if cs == 2
                                                       else "icv_igemm_smem<bf16,dense>")
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(p.in_channels, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    assert_bf16_close(y.reshape(-1, p.out_channels), ref.reshape(-1, p.out_channels))
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y.tobytes() == y_gather.tobytes()


def test_dense_a_pairs_chosen_by_k_loop_length():
    """Default plan (dense_cs = 0): CTA pairs from four 128-byte channel
    blocks up (the filter re-stream dominates the fill), single CTAs below;
    both equal the gather kernel bit for bit."""
    for c, want in ((64, "icv_igemm_smem<bf16,dense>"), (128, "icv_igemm_smem<bf16,dense>"),
                    (256, "icv_igemm_smem<bf16,dense,pair>"), (512, "icv_igemm_smem<bf16,dense,pair>")):
        g = dict(c=c, k=128, n=3, h=14, w=14)
        p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(g, True, torch.int64)
        assert L.kernel_name(p, shape, torch.bfloat16) == want
        y = icv.indirect_conv(x, pf, ib, p, tile).numpy()
        y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
        assert y.tobytes() == y_gather.tobytes()


def test_dense_a_offset_input_view():
    """An input that starts 16 bytes into its allocation still takes the TMA
    path (16-byte aligned base); the result equals the gather kernel's."""
    g = DENSE_GEOMS[0]
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(g, True, torch.int64)
    buf = torch.empty(x.data.numel() + 8, dtype=torch.bfloat16, device=DEV)
    buf[8:].copy_(x.data)
    xv = icv.NhwcTensor(shape, buf[8:])
    ibv = icv.init_indirection_buffer(xv, zero, p, o, tile, per_image=True)
    y = icv.indirect_conv(xv, pf, ibv, p, tile).numpy()
    assert y.tobytes() == icv.indirect_conv(x, pf, ib, p, tile).numpy().tobytes()


@pytest.mark.parametrize("geom", [dict(c=256, k=256, n=2, h=14, w=14), dict(c=48, k=40, n=3, h=5, w=7)])
def test_dense_a_u8_bit_exact(geom):
    g = dict(geom)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    assert L.kernel_name(p, shape, torch.uint8).startswith("icv_igemm_smem<u8,dense")
    rng = np.random.default_rng(7)
    xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
    wh = rng.integers(0, 256, p.out_channels * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
    qp = icv.QuantParams(128, 0.02, 127, 0.005, 128, 0.1)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, 1, 1, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=128)
    o = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, o, tile)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oq.indirect_conv_u8(xh, zero.cpu().numpy(), ib.offsets_host(), p, wh, bias, n, o.h, o.w,
                              128, 0.02, 127, 0.005, 128, 0.1)
    assert np.array_equal(y, ref), int((y != ref).sum())
    y_gather = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy().reshape(-1, p.out_channels)
    assert np.array_equal(y, y_gather)


def test_misaligned_tensors_fail_cleanly():
    """A tensor-core call on a 16-byte misaligned input raises
    UnsupportedError instead of faulting (the context stays usable)."""
    g = DENSE_GEOMS[0]
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(g, True, torch.int64)
    buf = torch.empty(x.data.numel() + 1, dtype=torch.bfloat16, device=DEV)
    xv = icv.NhwcTensor(shape, buf[1:])
    ibv = icv.init_indirection_buffer(xv, zero, p, o, tile, per_image=True)
    with pytest.raises(icv.UnsupportedError):
        icv.indirect_conv(xv, pf, ibv, p, tile)
    torch.cuda.synchronize()
    assert icv.indirect_conv(x, pf, ib, p, tile).numpy().shape[0] == o.numel


@pytest.mark.parametrize("cs", [1, 2])
@pytest.mark.parametrize("geom", [dict(c=128, k=512, n=64, h=28, w=28),    # 3 stages, 8 epilogue warps, 2 N tiles
                                  dict(c=1024, k=256, n=64, h=14, w=14),   # 16 K blocks per tile
                                  dict(c=64, k=64, n=64, h=56, w=56)])     # ~42 tiles per CTA
def test_dense_a_many_tiles_per_cta_equals_gather(geom, cs, tune):
    """Full-size ResNet-50 1x1 shapes: every CTA runs many tiles, so the
    stage ring wraps many times under several TMA issuers; the output must
    equal the IB-gather kernel's byte for byte."""
    tune(dense_cs=cs)
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom, True, torch.int64)
    y = icv.indirect_conv(x, pf, ib, p, tile)
    yg = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather")
    assert torch.equal(y.data, yg.data)


@pytest.mark.parametrize("wide", [0, 1])
@pytest.mark.parametrize("geom", [dict(c=64, k=256, n=2, h=14, w=14), dict(c=128, k=512, n=8, h=28, w=28),
                                  dict(c=72, k=200, n=1, h=9, w=7), dict(c=256, k=128, n=3, h=14, w=14)])
def test_epilogue_chunk_width_bit_identical(geom, wide, tune):
    """The 64-column epilogue (one 4 KB TMA box per chunk) and the 32-column
    one store the same bytes (same fp32 sums, same rounding); ragged K tails
    are clipped by TMA in both."""
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom, True, torch.int64)
    tune(epi_wide=0)
    y0 = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    g0 = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    tune(epi_wide=wide)
    y1 = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    g1 = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y0.tobytes() == y1.tobytes() and g0.tobytes() == g1.tobytes()
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(p.in_channels, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, shape.n, o.h, o.w)
    assert_bf16_close(y1.reshape(-1, p.out_channels), ref.reshape(-1, p.out_channels))


@pytest.mark.parametrize("geom", [dict(c=512, k=512, n=4, h=7, w=7), dict(c=128, k=256, n=2, h=9, w=9)])
def test_half_width_tiles_on_a_block256_packing(geom, tune):
    """BLOCK_N 128 tiles (chosen when BLOCK_N 256 would leave a partial last
    wave) read the BLOCK_N-256 packed filter unchanged: same sums, same bytes
    for the dense and the gather kernels."""
    p, shape, xh, wh, bias, x, pf, zero, ib, tile, o = _case(geom, True, torch.int64)
    tune(small_tile_bn=0)
    y0 = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    g0 = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    tune(small_tile_bn=100000)
    y1 = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    g1 = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy()
    assert y0.tobytes() == y1.tobytes() and g0.tobytes() == g1.tobytes()
