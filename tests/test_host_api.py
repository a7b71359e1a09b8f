"""Host-side logic of the drop-in API on the CPU: the same argument
validation and error types as the reference (/root/reference/pkg/src/
convbench/{tensors,indirect,gemm}.py), raised before any device work; and
no silent CPU fallback (CPU tensors are refused with NativeLibraryError)."""

import dataclasses

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from oracle import ib as oib


# ----------------------------------------------------------- tensors.py parity
def test_shape4_validation():
    with pytest.raises(ValueError):
        icv.Shape4(0, 1, 1, 1)
    with pytest.raises(ValueError):
        icv.Shape4(1, 1, 1.5, 1)
    assert icv.Shape4(2, 3, 4, 5).numel == 120


def test_conv_params_validation():
    with pytest.raises(ValueError):
        icv.ConvParams(kernel_h=0, kernel_w=1)
    with pytest.raises(ValueError):
        icv.ConvParams(kernel_h=1, kernel_w=1, pad_top=-1)
    p = make_params(r=3, s=2, c=4, k=5)
    assert p.kernel_elems == 6 and p.reduction_len == 24
    assert make_params().is_pointwise_unit_stride()
    assert not make_params(pt=1).is_pointwise_unit_stride()


def test_conv_output_shape_matches_oracle_and_enumeration(golden):
    for row in golden["ib_sweep"]:
        pd = row["params"]
        p = icv.ConvParams(**pd)
        shape = icv.Shape4(*row["in_shape"])
        out = icv.conv_output_shape(p, shape)
        assert (out.h, out.w) == tuple(row["out_hw"]) == oib.out_hw(p, shape.h, shape.w)


def test_conv_output_shape_errors():
    with pytest.raises(icv.InvalidGeometryError):
        icv.conv_output_shape(make_params(r=5, s=5, c=1), icv.Shape4(1, 3, 3, 1))
    with pytest.raises(ValueError):
        icv.conv_output_shape(make_params(c=2), icv.Shape4(1, 3, 3, 3))
    assert issubclass(icv.InvalidGeometryError, ValueError)
    assert issubclass(icv.StaleBufferError, RuntimeError)


def test_seeded_fills_match_reference_streams():
    t = icv.tensor_fill_random(icv.Shape4(1, 2, 3, 4), 7, device="cpu")
    want = np.random.default_rng(7).uniform(-1.0, 1.0, 24).astype(np.float32)
    assert np.array_equal(t.numpy(), want)
    f = icv.filter_fill_random(make_params(r=3, s=3, c=2, k=3), 8, device="cpu")
    assert np.array_equal(f.data.numpy(), np.random.default_rng(8).uniform(-1.0, 1.0, 54).astype(np.float32))
    assert icv.tensor_fill_sequential(icv.Shape4(1, 1, 2, 2), device="cpu").numpy().tolist() == [0, 1, 2, 3]


def test_nhwc_tensor_validation():
    with pytest.raises(TypeError):
        icv.NhwcTensor(icv.Shape4(1, 1, 1, 2), torch.zeros(2, dtype=torch.float64))
    with pytest.raises(ValueError):
        icv.NhwcTensor(icv.Shape4(1, 1, 1, 2), torch.zeros(3))
    with pytest.raises(ValueError):
        icv.NhwcTensor(icv.Shape4(1, 1, 2, 2), torch.zeros(2, 2))
    t = icv.NhwcTensor.from_array(np.arange(8, dtype=np.float32).reshape(1, 2, 2, 2), device="cpu")
    assert t.pixel_offset(0, 1, 1) == 6
    assert t.view4d().shape == (1, 2, 2, 2)


# ---------------------------------------------------------- indirect.py parity
def test_make_zero_row():
    with pytest.raises(ValueError):
        icv.make_zero_row(0, device="cpu")
    z = icv.make_zero_row(5, dtype=torch.uint8, device="cpu", fill=128)
    assert z.tolist() == [128] * 5


def _cpu_problem(c=3):
    p = make_params(r=3, s=3, pt=1, pl=1, c=c, k=4)
    x = icv.tensor_fill_random(icv.Shape4(2, 5, 5, c), 1, device="cpu")
    return p, x, icv.make_zero_row(c, device="cpu"), icv.conv_output_shape(p, x.shape)


def test_init_validation_precedes_device_work():
    p, x, zero, out_shape = _cpu_problem()
    tile = icv.TileConfig()
    with pytest.raises(ValueError):                                  # indirect.py:143-145
        icv.init_indirection_buffer(x, zero, p, icv.Shape4(2, 4, 5, 4), tile)
    with pytest.raises(ValueError):                                  # :146-147 (dtype)
        icv.init_indirection_buffer(x, zero.to(torch.bfloat16), p, out_shape, tile)
    with pytest.raises(ValueError):                                  # :146-147 (length)
        icv.init_indirection_buffer(x, icv.make_zero_row(2, device="cpu"), p, out_shape, tile)
    for bad in (0, 3):                                               # :148-150
        with pytest.raises(ValueError):
            icv.init_indirection_buffer(x, zero, p, out_shape, tile, batch=bad)
    with pytest.raises(icv.NativeLibraryError):                      # no CPU fallback
        icv.init_indirection_buffer(x, zero, p, out_shape, tile)


def _fake_ib(p, x, zero, out_shape, mr=4, batch=None):
    """A buffer assembled from the oracle's offsets (CPU), to exercise the
    stale-binding checks of indirect_conv without a device."""
    batch = x.shape.n if batch is None else batch
    offs = oib.compute_offsets(x.shape.astuple(), p, out_shape.h, out_shape.w, batch, mr)
    return icv.IndirectionBuffer(mr, batch, out_shape.h, out_shape.w, p, x.shape, x.data, zero,
                                 torch.from_numpy(offs))


def _fake_pf(p, nr=8, dtype=torch.float32):
    return icv.PackedFilter(p.out_channels, p.kernel_elems, p.in_channels, nr, dtype, p,
                            torch.zeros(16, dtype=torch.uint8), torch.zeros(p.out_channels))


def test_indirect_conv_stale_and_argument_checks():
    p, x, zero, out_shape = _cpu_problem()
    ib = _fake_ib(p, x, zero, out_shape)
    pf = _fake_pf(p)
    tile = icv.TileConfig()
    other = icv.tensor_fill_random(x.shape, 99, device="cpu")
    with pytest.raises(icv.StaleBufferError):                        # indirect.py:254-257
        icv.indirect_conv(other, pf, ib, p, tile)
    shifted = make_params(r=3, s=3, pt=1, pl=1, sy=2, sx=2, c=3, k=4)
    with pytest.raises(icv.StaleBufferError):                        # :258-259
        icv.indirect_conv(x, _fake_pf(shifted), ib, shifted, tile)
    with pytest.raises(icv.StaleBufferError):                        # :262-263 (mr)
        icv.indirect_conv(x, pf, ib, p, icv.TileConfig(mr=2, nr=8))
    with pytest.raises(icv.StaleBufferError):                        # :262-263 (nr)
        icv.indirect_conv(x, _fake_pf(p, nr=4), ib, p, tile)
    with pytest.raises(ValueError):                                  # :265-270
        icv.indirect_conv(x, pf, ib, p, tile, batch=3)
    bad_pf = dataclasses.replace(pf, k_out=5)
    with pytest.raises(ValueError):                                  # im2col.py:150-156
        icv.indirect_conv(x, bad_pf, ib, p, tile)
    # same shape, different binding object with the same storage is NOT stale
    same_storage = icv.NhwcTensor(x.shape, x.data.view(-1))
    with pytest.raises(icv.NativeLibraryError):                      # passes the checks, then: no CPU path
        icv.indirect_conv(same_storage, pf, ib, p, tile)


def test_update_for_batch_growth_checks():
    p, x, zero, out_shape = _cpu_problem()
    ib = _fake_ib(p, x, zero, out_shape, batch=2)
    assert icv.update_for_batch_growth(ib, 2) is ib                  # indirect.py:182-183
    with pytest.raises(ValueError):                                  # :175-179
        icv.update_for_batch_growth(ib, 1)
    with pytest.raises(ValueError):                                  # :180-181
        icv.update_for_batch_growth(ib, 3)


def test_rebind_shape_change_rejected():
    p, x, zero, out_shape = _cpu_problem()
    ib = _fake_ib(p, x, zero, out_shape)
    taller = icv.tensor_fill_random(icv.Shape4(2, 6, 5, 3), 2, device="cpu")
    with pytest.raises(ValueError):                                  # indirect.py:203-207
        icv.rebind_input(ib, taller, zero)


def test_buffer_properties_and_dereference():
    p, x, zero, out_shape = _cpu_problem()
    ib = _fake_ib(p, x, zero, out_shape, mr=4)
    pixels = 2 * 5 * 5
    assert ib.pixel_count == pixels
    assert ib.tile_count == -(-pixels // 4)
    assert ib.entry_count == ib.tile_count * 9 * 4
    assert ib.allocated_bytes == ib.entry_count * 8
    rows = ib.rows_for_tile(0)
    assert len(rows) == 9 * 4
    assert rows[0] is zero                                           # pixel (0,0,0), tap (0,0) is padding
    assert torch.equal(rows[4 * 4], x.data[0:3])                     # centre tap of pixel 0


# -------------------------------------------------------------- gemm.py parity
def test_tile_config_validation():
    with pytest.raises(ValueError):
        icv.TileConfig(mr=0)
    assert icv.TileConfig() == icv.TileConfig(4, 8)


def test_pack_filter_checks():
    p = make_params(r=3, s=3, c=3, k=4)
    filt = icv.filter_fill_random(p, 1, device="cpu")
    with pytest.raises(ValueError):                                  # gemm.py:145-146
        icv.pack_filter(filt, None, make_params(r=3, s=3, c=3, k=5), icv.TileConfig())
    with pytest.raises(ValueError):                                  # :164-165
        icv.pack_filter(filt, torch.zeros(4, dtype=torch.float64), p, icv.TileConfig())
    with pytest.raises(ValueError):
        icv.pack_filter(filt, torch.zeros(3), p, icv.TileConfig())
    with pytest.raises(ValueError):                                  # uint8 needs quantization params
        icv.pack_filter(icv.FilterTensor(4, 3, 3, 3, torch.zeros(108, dtype=torch.uint8)), None, p,
                        icv.TileConfig())
    with pytest.raises(icv.NativeLibraryError):                      # no CPU packing path
        icv.pack_filter(filt, None, p, icv.TileConfig())


def test_padded_bias_layout():
    p = make_params(c=2, k=5)
    pf = icv.PackedFilter(5, 1, 2, 4, torch.float32, p, torch.zeros(1, dtype=torch.uint8),
                          torch.arange(5, dtype=torch.float32))
    pb = pf.padded_bias()                                            # gemm.py:128-132
    assert pb.shape == (2, 4)
    assert pb.reshape(-1).tolist() == [0, 1, 2, 3, 4, 0, 0, 0]
