"""Parity of the CUDA path (through libicv.so's C ABI) with the oracle and
with the reference-generated golden fixtures.  Runs on a B200 only.

  * indirection buffer: bit-exact (int64 canonical form and int32)
  * float32 convolution: bit-exact (reference arithmetic contract)
  * bfloat16 convolution: rel 1e-2 vs the f32 oracle on bf16-rounded operands
  * uint8 convolution: bit-exact vs the int64 oracle
"""

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import P, make_params
from helpers import assert_bf16_close, fill_uniform, sha
from oracle import conv as oconv
from oracle import ib as oib
from oracle import quant as oq
from paper_1907_02129_b200 import _lib as L
from paper_1907_02129_b200.workloads import CFG1, CFG2, CFG3A, CFG3B, CFG4

pytestmark = pytest.mark.gpu
DEV = "cuda"


def to_params(d) -> icv.ConvParams:
    return icv.ConvParams(**d)


def dev_ib(params, shape, mr, batch=None, index_dtype=torch.int64, seed=0, dtype=torch.float32):
    x = icv.tensor_fill_random(shape, seed, device=DEV, dtype=dtype)
    zero = icv.make_zero_row(params.in_channels, dtype=dtype, device=DEV)
    out_shape = icv.conv_output_shape(params, shape)
    ib = icv.init_indirection_buffer(x, zero, params, out_shape, icv.TileConfig(mr=mr), batch=batch,
                                     index_dtype=index_dtype)
    return x, zero, out_shape, ib


# --------------------------------------------------------------------- IB (K1)
def test_ib_known_answers(golden):
    for case in golden["ib_kat"]:
        p = to_params(case["params"])
        shape = icv.Shape4(*case["in_shape"])
        _, _, _, ib = dev_ib(p, shape, case["mr"])
        got = ib.offsets_host()
        assert list(got.shape) == case["offsets_shape"], case["name"]
        assert got.reshape(-1).tolist() == case["offsets"], case["name"]


def test_ib_sweep_digests_int64_and_int32(golden):
    for row in golden["ib_sweep"]:
        p = to_params(row["params"])
        shape = icv.Shape4(*row["in_shape"])
        for mr, (oshape, digest) in row["mr"].items():
            _, _, _, ib = dev_ib(p, shape, int(mr))
            assert sha(ib.offsets_host().astype("<i8")) == digest, (row["i"], mr)
            if mr == "4":
                _, _, _, ib32 = dev_ib(p, shape, 4, index_dtype=torch.int32)
                assert ib32.offsets.dtype == torch.int32
                assert sha(ib32.offsets_host().astype("<i8")) == digest, (row["i"], "int32")
        if "batch1_mr4" in row:
            x, zero, out_shape, ib1 = dev_ib(p, shape, 4, batch=1)
            assert sha(ib1.offsets_host().astype("<i8")) == row["batch1_mr4"][1]
            grown = icv.update_for_batch_growth(ib1, 2)
            assert sha(grown.offsets_host().astype("<i8")) == row["grown_mr4"]


def test_ib_matches_oracle_at_full_config_sizes():
    """Every BASELINE config, canonical int64 form, bit-exact (cfg3a's IB is
    19.7 M entries at mr=128)."""
    for w in (CFG1, CFG2, CFG3A, CFG3B, CFG4):
        for mr in (4, 128):
            x = icv.NhwcTensor.empty(w.in_shape, dtype=torch.uint8 if w.dtype == "u8" else torch.bfloat16,
                                     device=DEV)
            zero = icv.make_zero_row(w.in_shape.c, dtype=x.dtype, device=DEV)
            out_shape = icv.conv_output_shape(w.params, w.in_shape)
            ib = icv.init_indirection_buffer(x, zero, w.params, out_shape, icv.TileConfig(mr=mr))
            oh, ow = w.out_hw
            want = oib.compute_offsets(w.in_shape.astuple(), w.params, oh, ow, w.in_shape.n, mr)
            assert np.array_equal(ib.offsets_host(), want), (w.name, mr)


def test_ib_growth_preserves_prefix_on_device():
    params = make_params(r=3, s=3, pt=1, pl=1, c=3, k=4)
    phys = icv.tensor_fill_random(icv.Shape4(2, 3, 3, 3), seed=50, device=DEV)
    zero = icv.make_zero_row(3, device=DEV)
    out1 = icv.conv_output_shape(params, phys.shape)
    ib1 = icv.init_indirection_buffer(phys, zero, params, out1, icv.TileConfig(), batch=1)
    grown = icv.update_for_batch_growth(ib1, 2)
    fresh = icv.init_indirection_buffer(phys, zero, params, out1, icv.TileConfig(), batch=2)
    assert torch.equal(grown.offsets, fresh.offsets)
    keep = ib1.pixel_count // 4
    assert torch.equal(grown.offsets[:keep], ib1.offsets[:keep])
    assert icv.update_for_batch_growth(grown, 2) is grown


# ------------------------------------------------------------ float32 (K5)
def run_f32(params, shape, seed_x, seed_w, bias, mr=4, nr=8):
    tile = icv.TileConfig(mr=mr, nr=nr)
    x = icv.NhwcTensor(shape, torch.from_numpy(fill_uniform(shape.numel, seed_x)).to(DEV))
    filt = icv.filter_fill_random(params, seed_w, device=DEV)
    zero = icv.make_zero_row(params.in_channels, device=DEV)
    out_shape = icv.conv_output_shape(params, shape)
    ib = icv.init_indirection_buffer(x, zero, params, out_shape, tile)
    pf = icv.pack_filter(filt, None if bias is None else torch.from_numpy(bias), params, tile)
    return icv.indirect_conv(x, pf, ib, params, tile).numpy()


def test_f32_sweep_bit_exact(golden):
    for row in golden["conv_sweep"]:
        p = to_params(row["params"])
        shape = icv.Shape4(*row["in_shape"])
        i = row["i"]
        bias = np.random.default_rng(i + 2).uniform(-1.0, 1.0, p.out_channels).astype(np.float32)
        out = run_f32(p, shape, i, i + 1, bias)
        assert sha(out.astype("<f4")) == row["out_sha"], (i, row["params"], row["in_shape"])


@pytest.mark.parametrize("mr", [None, 1, 128])
def test_f32_kat_bit_exact(golden, mr):
    for row in golden["conv_kat"]:
        p = to_params(row["params"])
        shape = icv.Shape4(*row["in_shape"])
        s = row["seed"]
        bias = np.random.default_rng(s + 2).uniform(-1, 1, p.out_channels).astype(np.float32)
        out = run_f32(p, shape, s, s + 1, bias, mr=row["mr"] if mr is None else mr, nr=row["nr"])
        assert sha(out.astype("<f4")) == row["out_sha"], row["name"]


def test_cfg1_bit_exact(golden):
    w = CFG1
    tile = icv.TileConfig()
    x = icv.NhwcTensor(w.in_shape, torch.from_numpy(w.input_host()).to(DEV))
    filt = icv.FilterTensor(64, 3, 3, 64, torch.from_numpy(w.filter_host()).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(w.bias_host()), w.params, tile)
    zero = icv.make_zero_row(64, device=DEV)
    ib = icv.init_indirection_buffer(x, zero, w.params, icv.conv_output_shape(w.params, w.in_shape), tile)
    assert sha(ib.offsets_host().astype("<i8")) == golden["cfg1"]["ib_mr4_sha"]
    out = icv.indirect_conv(x, pf, ib, w.params, tile).numpy()
    assert sha(out.astype("<f4")) == golden["cfg1"]["out_sha"]


# ------------------------------------------------------------ bfloat16 (K2)
def bf16_problem(w, n_img=None, mr=128, index_dtype=torch.int64):
    n_img = w.in_shape.n if n_img is None else n_img
    shape = icv.Shape4(n_img, w.in_shape.h, w.in_shape.w, w.in_shape.c)
    xh = w.input_host(0, n_img)
    wh = w.filter_host()
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    p = w.params
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                            torch.from_numpy(wh).to(DEV).to(torch.bfloat16))
    tile = icv.TileConfig(mr=mr)
    pf = icv.pack_filter(filt, None, p, tile)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), tile, index_dtype=index_dtype)
    y = icv.indirect_conv(x, pf, ib, p, tile)
    return shape, oconv.bf16_round(xh), oconv.bf16_round(wh), ib, y


@pytest.mark.parametrize("w", [CFG2, CFG3A, CFG3B], ids=lambda w: w.name)
def test_bf16_slice_vs_reference_golden(golden, w):
    """N=1 slices whose f32-reference outputs are pinned in the fixtures."""
    case = next(c for c in golden["bf16_slices"] if c["name"] == w.name)
    shape, xr, wr, ib, y = bf16_problem(w, n_img=case["images"])
    assert sha(xr.astype("<f4")) == case["x_bf16_sha"]
    oh, ow = w.out_hw
    ref = oconv.indirect_conv_f32(xr, np.zeros(shape.c, np.float32), ib.offsets_host(), w.params, wr, None,
                                  shape.n, oh, ow)
    assert sha(ref.astype("<f4")) == case["out_sha"]          # oracle == reference on these operands
    assert_bf16_close(y.numpy().reshape(ref.shape), ref)


@pytest.mark.parametrize("w", [CFG2, CFG3A, CFG3B], ids=lambda w: w.name)
def test_bf16_full_config_sampled_pixels(w):
    """Full BASELINE batch; the oracle is evaluated on 4096 seeded random
    output pixels (rows are independent) plus the first and last pixel."""
    shape, xr, wr, ib, y = bf16_problem(w)
    oh, ow = w.out_hw
    pixels = shape.n * oh * ow
    idx = np.unique(np.concatenate([[0, pixels - 1], np.random.default_rng(7).integers(0, pixels, 4096)]))
    ref = oconv.indirect_conv_f32(xr, np.zeros(shape.c, np.float32), ib.offsets_host(), w.params, wr, None,
                                  shape.n, oh, ow, pixel_index=idx)
    got = y.numpy().reshape(pixels, -1)[idx]
    assert_bf16_close(got, ref)


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=64, k=64, n=2, h=9, w=11, mr=4),       # K=64 tile, tails
    dict(r=3, s=3, pt=1, pl=1, c=72, k=200, n=1, h=13, w=7, mr=3),      # C % 64 != 0, K % BN != 0
    dict(r=1, s=1, c=256, k=512, n=3, h=7, w=7, mr=128),                # pointwise, 2 N tiles
    dict(r=3, s=2, sy=2, sx=1, dy=2, dx=1, pt=2, pl=1, pb=0, pr=2, c=16, k=40, n=2, h=10, w=9, mr=1),
    dict(r=5, s=5, pt=2, pl=2, c=8, k=24, n=1, h=6, w=6, mr=4),         # C=8: single 16-byte chunk
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=2, h=20, w=18, mr=4),   # channel-poor stem (tcgen05)
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=100, n=1, h=15, w=17, mr=128),  # stem, K tail in a 128 tile
    dict(r=3, s=3, pt=1, pl=1, c=3, k=24, n=3, h=9, w=11, mr=3),        # 3x3 first layer, K < tile
    dict(r=3, s=3, sy=2, sx=2, pt=0, pl=1, pb=2, pr=0, c=1, k=40, n=2, h=13, w=10, mr=1),   # C=1
    dict(r=5, s=5, pt=2, pl=2, c=5, k=16, n=1, h=8, w=8, mr=4),         # channel-poor, CUDA-core variant
])
@pytest.mark.parametrize("index_dtype", [torch.int64, torch.int32])
def test_bf16_edge_geometries(geom, index_dtype):
    g = dict(geom)
    n, h, wd, mr = g.pop("n"), g.pop("h"), g.pop("w"), g.pop("mr")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(3)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=mr)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, index_dtype=index_dtype)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(shape.c, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, n, out_shape.h, out_shape.w)
    assert_bf16_close(y, ref)


# --------------------------------------------------------------- uint8 (K3)
def u8_problem(w, n_img=None, mr=4):
    n_img = w.in_shape.n if n_img is None else n_img
    shape = icv.Shape4(n_img, w.in_shape.h, w.in_shape.w, w.in_shape.c)
    q = w.quant
    qp = icv.QuantParams(q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                         q.output_zero_point, q.output_scale, q.output_min, q.output_max)
    xh = w.input_host(0, n_img)
    wh = w.filter_host()
    bias = w.bias_host()
    p = w.params
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    tile = icv.TileConfig(mr=mr)
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=q.input_zero_point)
    ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), tile)
    y = icv.indirect_conv(x, pf, ib, p, tile)
    return shape, xh, wh, bias, zero.cpu().numpy(), ib, y


def test_u8_cfg4_full_batch_bit_exact_sampled():
    w = CFG4
    q = w.quant
    shape, xh, wh, bias, zero, ib, y = u8_problem(w)
    oh, ow = w.out_hw
    pixels = shape.n * oh * ow
    idx = np.unique(np.concatenate([[0, pixels - 1], np.random.default_rng(8).integers(0, pixels, 3000)]))
    ref = oq.indirect_conv_u8(xh, zero, ib.offsets_host(), w.params, wh, bias, shape.n, oh, ow,
                              q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                              q.output_zero_point, q.output_scale, pixel_index=idx)
    got = y.numpy().reshape(pixels, -1)[idx]
    assert np.array_equal(got, ref), int((got != ref).sum())


def test_u8_cfg4_slice_bit_exact_all_pixels():
    w = CFG4
    q = w.quant
    shape, xh, wh, bias, zero, ib, y = u8_problem(w, n_img=2, mr=128)
    oh, ow = w.out_hw
    ref = oq.indirect_conv_u8(xh, zero, ib.offsets_host(), w.params, wh, bias, shape.n, oh, ow,
                              q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                              q.output_zero_point, q.output_scale)
    assert np.array_equal(y.numpy().reshape(ref.shape), ref)


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=16, k=24, n=2, h=7, w=9, mr=4, zx=3, zw=250),
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=48, k=130, n=1, h=11, w=10, mr=1, zx=128, zw=127),
    dict(r=1, s=1, c=128, k=64, n=2, h=5, w=5, mr=128, zx=0, zw=0),
    dict(r=3, s=3, pt=1, pl=1, c=5, k=9, n=1, h=6, w=5, mr=4, zx=100, zw=7),     # C % 16 != 0 (CUDA cores)
])
def test_u8_edge_geometries(geom):
    g = dict(geom)
    n, h, wd, mr, zx, zw = (g.pop(k) for k in ("n", "h", "w", "mr", "zx", "zw"))
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(9)
    xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
    wh = rng.integers(0, 256, p.out_channels * p.kernel_elems * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
    qp = icv.QuantParams(zx, 0.02, zw, 0.005, 128, 0.1)
    tile = icv.TileConfig(mr=mr)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=zx)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oq.indirect_conv_u8(xh, zero.cpu().numpy(), ib.offsets_host(), p, wh, bias, n, out_shape.h,
                              out_shape.w, zx, 0.02, zw, 0.005, 128, 0.1)
    assert np.array_equal(y, ref), int((y != ref).sum())


def test_requant_params_native_equals_oracle():
    for sx, sw, so in [(0.02, 0.005, 0.1), (0.5, 0.25, 0.3), (1e-3, 2e-3, 7e-4), (0.9, 0.9, 0.95)]:
        qp = icv.QuantParams(0, sx, 0, sw, 0, so)
        assert qp.requant() == oq.requant_params(sx, sw, so)


# ------------------------------------------------------- API semantics on GPU
def test_api_semantics_mirror_reference_tests():
    """test_indirect.py:184-216 and :293-305 on the device path."""
    params = make_params(r=3, s=3, pt=1, pl=1, c=3, k=4)
    tile = icv.TileConfig()
    x = icv.tensor_fill_random(icv.Shape4(2, 5, 5, 3), 15, device=DEV)
    zero = icv.make_zero_row(3, device=DEV)
    out_shape = icv.conv_output_shape(params, x.shape)
    ib = icv.init_indirection_buffer(x, zero, params, out_shape, tile)
    pf = icv.pack_filter(icv.filter_fill_random(params, 16, device=DEV), None, params, tile)
    a = icv.indirect_conv(x, pf, ib, params, tile).numpy()
    b = icv.indirect_conv(x, pf, ib, params, tile).numpy()
    assert a.tobytes() == b.tobytes()                                 # repeat invocations identical
    assert zero.cpu().tolist() == [0.0, 0.0, 0.0]                     # zero row stays pure
    small = icv.indirect_conv(x, pf, ib, params, tile, batch=1)       # logical truncation
    assert small.shape.n == 1
    assert small.numpy().tobytes() == a[: 5 * 5 * 4].tobytes()
    other = icv.tensor_fill_random(x.shape, 999, device=DEV)
    with pytest.raises(icv.StaleBufferError):
        icv.indirect_conv(other, pf, ib, params, tile)
    with pytest.raises(icv.StaleBufferError):
        icv.indirect_conv(x, pf, ib, params, icv.TileConfig(mr=2, nr=8))
    shifted = make_params(r=3, s=3, pt=1, pl=1, sy=2, sx=2, c=3, k=4)
    pf2 = icv.pack_filter(icv.filter_fill_random(shifted, 1, device=DEV), None, shifted, tile)
    with pytest.raises(icv.StaleBufferError):
        icv.indirect_conv(x, pf2, ib, shifted, tile)
    with pytest.raises(ValueError):
        icv.indirect_conv(x, pf, ib, params, tile, batch=3)
    # rebind to a copy gives the same numbers; same object -> identical buffer
    copy = icv.tensor_fill_random(x.shape, 15, device=DEV)
    ib2 = icv.rebind_input(ib, copy, icv.make_zero_row(3, device=DEV))
    assert torch.equal(ib2.offsets, ib.offsets)
    assert icv.indirect_conv(copy, pf, ib2, params, tile).numpy().tobytes() == a.tobytes()
    with pytest.raises(ValueError):
        icv.rebind_input(ib, icv.tensor_fill_random(icv.Shape4(2, 6, 5, 3), 1, device=DEV), zero)


def test_grown_buffer_convolves_like_fresh():
    """test_indirect.py:279-291 (bit-exact vs the direct oracle)."""
    params = make_params(r=3, s=3, pt=1, pl=1, c=3, k=5)
    tile = icv.TileConfig()
    phys = icv.tensor_fill_random(icv.Shape4(2, 4, 4, 3), 53, device=DEV)
    zero = icv.make_zero_row(3, device=DEV)
    out_shape = icv.conv_output_shape(params, phys.shape)
    pf = icv.pack_filter(icv.filter_fill_random(params, 54, device=DEV), None, params, tile)
    ib1 = icv.init_indirection_buffer(phys, zero, params, out_shape, tile, batch=1)
    out = icv.indirect_conv(phys, pf, icv.update_for_batch_growth(ib1, 2), params, tile).numpy()
    ref = oconv.direct_conv_f32(fill_uniform(phys.shape.numel, 53).reshape(2, 4, 4, 3),
                                fill_uniform(5 * 9 * 3, 54), None, params)
    assert out.tobytes() == ref.reshape(-1).tobytes()


def test_kernel_selection_is_native_tensor_core_for_baseline_configs():
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16).startswith("icv_igemm_")
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16).endswith("<bf16>")
    assert L.kernel_name(CFG3B.params, CFG3B.in_shape, torch.bfloat16).startswith("icv_igemm_")
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8).startswith("icv_igemm_")
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8).startswith("icv_igemm_smem<u8")
    assert L.kernel_name(CFG1.params, CFG1.in_shape, torch.float32) == "icv_conv_f32_exact"
    before = L.launch_count()
    bf16_problem(CFG2, n_img=1)
    assert L.launch_count() > before


# ------------------------------------------------- per-image (batch-invariant) IB
def test_per_image_ib_expands_to_canonical(golden):
    for row in golden["ib_sweep"][::5]:
        p = to_params(row["params"])
        shape = icv.Shape4(*row["in_shape"])
        for mr, (oshape, digest) in row["mr"].items():
            x = icv.tensor_fill_random(shape, 0, device=DEV)
            zero = icv.make_zero_row(p.in_channels, device=DEV)
            ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), icv.TileConfig(mr=int(mr)),
                                             per_image=True, index_dtype=torch.int32)
            assert ib.offsets.shape[0] == -(-(ib.out_h * ib.out_w) // int(mr))
            assert sha(ib.offsets_host().astype("<i8")) == digest, (row["i"], mr)


@pytest.mark.parametrize("w", [CFG1, CFG2, CFG3A, CFG3B, CFG4], ids=lambda w: w.name)
def test_per_image_ib_gives_identical_outputs(w):
    """Same bytes out of every kernel family whichever buffer form it reads
    (2 images of each config; the stem reads 157 MB less with per-image)."""
    n = 2
    w = w.with_batch(max(n, w.in_shape.n))
    shape = icv.Shape4(n, w.in_shape.h, w.in_shape.w, w.in_shape.c)
    p = w.params
    dt = {"f32": torch.float32, "bf16": torch.bfloat16, "u8": torch.uint8}[w.dtype]
    x = icv.NhwcTensor(shape, torch.from_numpy(w.input_host(0, n)).to(DEV).to(dt))
    qp, fill = None, 0
    if w.quant is not None:
        q = w.quant
        qp = icv.QuantParams(q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                             q.output_zero_point, q.output_scale)
        fill = q.input_zero_point
    bias = w.bias_host()
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                            torch.from_numpy(w.filter_host()).to(DEV).to(dt))
    outs = []
    for mr in (4, 128):
        tile = icv.TileConfig(mr=mr)
        pf = icv.pack_filter(filt, None if bias is None else torch.from_numpy(bias), p, tile, quant=qp)
        zero = icv.make_zero_row(p.in_channels, dtype=dt, device=DEV, fill=fill)
        for per_image in (False, True):
            ib = icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, shape), tile, per_image=per_image)
            outs.append(icv.indirect_conv(x, pf, ib, p, tile).data.clone())
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_per_image_growth_needs_no_rebuild():
    p = make_params(r=3, s=3, pt=1, pl=1, c=8, k=8)
    x = icv.tensor_fill_random(icv.Shape4(3, 5, 6, 8), 3, device=DEV, dtype=torch.bfloat16)
    zero = icv.make_zero_row(8, dtype=torch.bfloat16, device=DEV)
    out_shape = icv.conv_output_shape(p, x.shape)
    ib1 = icv.init_indirection_buffer(x, zero, p, out_shape, icv.TileConfig(), batch=1, per_image=True)
    grown = icv.update_for_batch_growth(ib1, 3)
    assert grown.offsets is ib1.offsets and grown.batch == 3
    fresh = icv.init_indirection_buffer(x, zero, p, out_shape, icv.TileConfig())
    assert np.array_equal(grown.offsets_host(), fresh.offsets_host())


@pytest.mark.parametrize("geom", [
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=5, h=32, w=32),    # Ho*Wo = 256: image-major schedule
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=4, h=30, w=26),    # tiles straddle images
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=128, n=3, h=64, w=32),   # 128-wide filter, image-major
    dict(r=3, s=3, pt=1, pl=1, c=1, k=40, n=7, h=16, w=8),                 # C = 1, image-major
    dict(r=3, s=3, pt=1, pl=1, c=3, k=32, n=2, h=200, w=190),              # wide rows
    dict(r=3, s=3, pt=1, pl=1, c=3, k=32, n=2, h=5, w=1500),               # window > 2048 pixels: global path
])
@pytest.mark.parametrize("index_dtype", [torch.int64, torch.int32])
def test_stem_per_image_schedules(geom, index_dtype):
    """Channel-poor kernel with a per-image buffer: pattern reuse across
    images (image-major schedule) and tiles straddling two images."""
    g = dict(geom)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(11)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    out_shape = icv.conv_output_shape(p, shape)
    assert L.kernel_name(p, shape, torch.bfloat16) in ("icv_igemm_stem<bf16>", "icv_igemm_rows<bf16>")
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, index_dtype=index_dtype, per_image=True)
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(shape.c, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, n, out_shape.h, out_shape.w)
    assert_bf16_close(y, ref)



# ----------------------------------------------- row-sliding stem kernel (K4b)
def _stem_problem(g, index_dtype=torch.int64, per_image=True, seed=13):
    g = dict(g)
    n, h, wd = g.pop("n"), g.pop("h"), g.pop("w")
    p = make_params(**g)
    shape = icv.Shape4(n, h, wd, p.in_channels)
    rng = np.random.default_rng(seed)
    xh = rng.standard_normal(shape.numel, dtype=np.float32)
    wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
    bias = rng.standard_normal(p.out_channels, dtype=np.float32)
    tile = icv.TileConfig(mr=128)
    x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
    filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
    pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
    zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
    out_shape = icv.conv_output_shape(p, shape)
    ib = icv.init_indirection_buffer(x, zero, p, out_shape, tile, index_dtype=index_dtype, per_image=per_image)
    return p, shape, xh, wh, bias, x, pf, ib, tile, out_shape


@pytest.mark.parametrize("geom", [
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=3, h=96, w=88),     # one tile per output row
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=2, h=70, w=320),    # two tiles per row (Wo = 160)
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=40, n=2, h=65, w=64),     # K < 64, odd H
    dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=128, n=1, h=64, w=96),    # 128-wide filter
    dict(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=3, k=64, n=2, h=80, w=72),     # 3x3/2 (one K step)
    dict(r=7, s=7, sy=2, sx=2, pt=2, pl=4, pb=4, pr=1, c=3, k=64, n=2, h=70, w=80),   # asymmetric padding
])
@pytest.mark.parametrize("per_image,index_dtype,rows_per_tile", [(True, torch.int64, "1"), (False, torch.int64, "1"),
                                                                 (True, torch.int32, "1"), (True, torch.int64, "2")])
def test_rows_kernel_matches_oracle(geom, per_image, index_dtype, rows_per_tile, tune):
    """rows_per_tile 2: the opt-in two-output-row tiles (ICV_ROWS_RP=2; BN 64
    filters only, others keep one row per tile)."""
    tune(rows_rp=int(rows_per_tile))
    p, shape, xh, wh, bias, x, pf, ib, tile, o = _stem_problem(geom, index_dtype, per_image)
    assert L.kernel_name(p, shape, torch.bfloat16) == "icv_igemm_rows<bf16>"
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    pixels = o.n * o.h * o.w
    idx = np.unique(np.concatenate([np.arange(min(pixels, 2 * o.w)), np.arange(max(0, pixels - 2 * o.w), pixels),
                                    np.random.default_rng(1).integers(0, pixels, 2048)]))
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(shape.c, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, o.n, o.h, o.w, pixel_index=idx)
    assert_bf16_close(y[idx], ref)


def test_rows_kernel_equals_tap_gather_and_respects_noncanonical_buffers():
    """The row-sliding kernel gives the tap-by-tap gather kernel's answer; a
    buffer that differs from the canonical one is detected by icv_ib_check
    and then read entry by entry (the kernel follows the buffer)."""
    g = dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64, n=2, h=64, w=64)
    p, shape, xh, wh, bias, x, pf, ib, tile, o = _stem_problem(g)
    assert ib.verify() == 0 and ib.canonical
    y_rows = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    ib.canonical = False
    y_gather = icv.indirect_conv(x, pf, ib, p, tile).numpy()
    assert_bf16_close(y_rows, y_gather)    # same sums, different fp32 accumulation order
    # redirect one tap of pixel 5 to another input row: the gather path follows it
    ib.offsets[0, 24, 5] = ib.offsets[0, 24, 9]
    assert ib.verify() > 0 and not ib.canonical
    y = icv.indirect_conv(x, pf, ib, p, tile).numpy().reshape(-1, p.out_channels)
    ref = oconv.indirect_conv_f32(oconv.bf16_round(xh), np.zeros(shape.c, np.float32), ib.offsets_host(), p,
                                  oconv.bf16_round(wh), bias, o.n, o.h, o.w, pixel_index=np.arange(16))
    assert_bf16_close(y[:16], ref)


@pytest.mark.parametrize("index_dtype", [torch.int64, torch.int32])
@pytest.mark.parametrize("per_image", [False, True])
def test_ib_check_accepts_built_buffers(index_dtype, per_image):
    for g in (dict(r=3, s=3, pt=1, pl=1, c=8, k=8, n=3, h=9, w=7), dict(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=64,
                                                                        n=2, h=40, w=48)):
        p, shape, xh, wh, bias, x, pf, ib, tile, o = _stem_problem(g, index_dtype, per_image)
        assert ib.verify() == 0
