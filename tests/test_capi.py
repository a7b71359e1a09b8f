"""The C-ABI library (libicv.so): loads without a GPU, exports every symbol
include/icv.h declares, and its host-only entry points (geometry, sizes,
requantization constants, kernel selection) agree with the oracle.  No
compute call is made here (CPU only)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, make_params
from oracle import ib as oib
from oracle import quant as oq
from paper_1907_02129_b200 import _lib as L

HEADER = os.path.join(ROOT, "include", "icv.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"ICV_API\s+[\w\s\*]+?\b(icv_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("icv_ib_build", "icv_conv", "icv_pack_filter", "icv_out_shape", "icv_last_error"):
        assert name in syms
    assert len(syms) >= 12


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # and the ctypes binding covers the whole declared surface
    assert set(declared_symbols()) <= set(L.SIGNATURES)


def test_abi_version():
    assert L.lib().icv_abi_version() == 2


def test_tuning_knobs_roundtrip_and_reject_unknown():
    assert L.get_tuning("win") == -1
    assert L.get_tuning("dense_a") == 1
    with L.tuning(win=0, win_cs=1):
        assert L.get_tuning("win") == 0 and L.get_tuning("win_cs") == 1
    assert L.get_tuning("win") == -1 and L.get_tuning("win_cs") == 2
    with pytest.raises(ValueError):
        L.set_tuning("no_such_knob", 1)


def test_kernel_selection_flags():
    import torch

    from paper_1907_02129_b200.workloads import CFG2, CFG3A, resnet50_layers

    # the IB-gather request turns off every canonical-buffer specialisation
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16) == "icv_igemm_win<bf16>"
    g = L.DEFAULT_FLAGS | L.ICV_PREFER_GATHER
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16, g) == "icv_igemm_smem<bf16>"
    assert L.kernel_name(CFG3A.params, CFG3A.in_shape, torch.bfloat16, g) == "icv_igemm_stem<bf16>"
    # a non-canonical buffer never takes the window / row / dense-A kernels
    nc = L.ICV_ZERO_ROW_ZEROS
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16, nc) == "icv_igemm_smem<bf16>"
    assert L.kernel_name(CFG3A.params, CFG3A.in_shape, torch.bfloat16, nc) == "icv_igemm_stem<bf16>"
    # 1x1 stride-1 layers: dense TMA rows unless the gather kernel is requested
    one = [(n, s, p) for n, s, p in resnet50_layers(8) if n == "s3b2_1x1a"][0]
    assert L.kernel_name(one[2], one[1], torch.bfloat16).startswith("icv_igemm_smem<bf16,dense")
    assert L.kernel_name(one[2], one[1], torch.bfloat16, g) == "icv_igemm_smem<bf16>"
    with L.tuning(dense_a=0):   # (without the dense boxes the im2col TMA tiles serve a long-K 1x1 as well)
        assert L.kernel_name(one[2], one[1], torch.bfloat16) == "icv_igemm_smem<bf16,im2col,pair>"
    with L.tuning(dense_a=0, im2col_a=0):
        assert L.kernel_name(one[2], one[1], torch.bfloat16) == "icv_igemm_smem<bf16>"


def _out_shape(params, shape):
    d, s, o = L.desc_of(params), L.Shape(*shape), L.Shape()
    st = L.lib().icv_out_shape(ctypes.byref(d), ctypes.byref(s), ctypes.byref(o))
    return st, (o.n, o.h, o.w, o.c)


def test_out_shape_matches_oracle_over_sweep(golden):
    for row in golden["ib_sweep"][::7]:
        p = make_params(r=row["params"]["kernel_h"], s=row["params"]["kernel_w"],
                        sy=row["params"]["stride_h"], sx=row["params"]["stride_w"],
                        dy=row["params"]["dilation_h"], dx=row["params"]["dilation_w"],
                        pt=row["params"]["pad_top"], pl=row["params"]["pad_left"],
                        c=row["params"]["in_channels"], k=row["params"]["out_channels"])
        st, out = _out_shape(p, row["in_shape"])
        assert st == 0
        assert (out[1], out[2]) == tuple(row["out_hw"])
        assert out == (row["in_shape"][0], *row["out_hw"], p.out_channels)


def test_out_shape_errors_map_to_reference_exceptions():
    p = make_params(r=3, s=3, c=4, k=2)
    st, _ = _out_shape(p, (1, 2, 2, 4))                        # 3x3 does not fit in 2x2 (tensors.py:203-208)
    assert st == L.ICV_ERR_GEOMETRY
    assert "does not fit" in L.last_error()
    st, _ = _out_shape(p, (1, 5, 5, 3))                        # channel mismatch (tensors.py:191-194)
    assert st == L.ICV_ERR_ARG
    with pytest.raises(ValueError):
        L.check(st, "x")
    from paper_1907_02129_b200.errors import InvalidGeometryError

    with pytest.raises(InvalidGeometryError):
        L.check(L.ICV_ERR_GEOMETRY, "x")


def test_ib_entries_formula():
    """entries = ceil(P/mr)*mr*RS (test_indirect.py:95-101)."""
    p = make_params(r=2, s=3, sy=2, sx=1, pt=1, pl=1, c=2)
    shape = (2, 7, 5, 2)
    oh, ow = oib.out_hw(p, 7, 5)
    for mr in (1, 3, 4, 128):
        for batch in (1, 2):
            t, e = ctypes.c_int64(), ctypes.c_int64()
            d, s = L.desc_of(p), L.Shape(*shape)
            assert L.lib().icv_ib_entries(ctypes.byref(d), ctypes.byref(s), batch, mr, ctypes.byref(t),
                                          ctypes.byref(e)) == 0
            pixels = batch * oh * ow
            assert t.value == -(-pixels // mr)
            assert e.value == t.value * mr * 6
    d, s = L.desc_of(p), L.Shape(*shape)
    assert L.lib().icv_ib_entries(ctypes.byref(d), ctypes.byref(s), 3, 4, None, None) == L.ICV_ERR_ARG


def test_requant_params_match_oracle():
    rng = np.random.default_rng(0)
    cases = [(0.02, 0.005, 0.1)] + [tuple(float(v) for v in rng.uniform(1e-3, 1.0, 3)) for _ in range(200)]
    for sx, sw, so in cases:
        m, sh = ctypes.c_int32(), ctypes.c_int32()
        st = L.lib().icv_requant_params(sx, sw, so, ctypes.byref(m), ctypes.byref(sh))
        try:
            want = oq.requant_params(sx, sw, so)
        except ValueError:
            assert st != 0
            continue
        assert st == 0
        assert (m.value, sh.value) == want, (sx, sw, so)


def test_packed_filter_bytes_and_kernel_selection():
    from paper_1907_02129_b200.workloads import CFG1, CFG2, CFG3A, CFG3B, CFG4

    for w, dt in ((CFG1, L.ICV_F32), (CFG2, L.ICV_BF16), (CFG3A, L.ICV_BF16), (CFG3B, L.ICV_BF16),
                  (CFG4, L.ICV_U8)):
        n = ctypes.c_int64()
        d = L.desc_of(w.params)
        assert L.lib().icv_packed_filter_bytes(ctypes.byref(d), dt, ctypes.byref(n)) == 0
        p = w.params
        assert n.value >= p.out_channels * p.kernel_elems * p.in_channels
    import torch

    assert L.kernel_name(CFG1.params, CFG1.in_shape, torch.float32) == "icv_conv_f32_exact"
    assert L.kernel_name(CFG2.params, CFG2.in_shape, torch.bfloat16).startswith("icv_igemm_")
    assert L.kernel_name(CFG3B.params, CFG3B.in_shape, torch.bfloat16).startswith("icv_igemm_")
    assert L.kernel_name(CFG4.params, CFG4.in_shape, torch.uint8).startswith("icv_igemm_")
    assert L.kernel_name(CFG3A.params, CFG3A.in_shape, torch.bfloat16) == "icv_igemm_rows<bf16>"   # C=3 stem


def test_null_and_range_arguments_are_rejected():
    p = make_params(r=3, s=3, pt=1, pl=1, c=8, k=8)
    d, s = L.desc_of(p), L.Shape(1, 4, 4, 8)
    lib = L.lib()
    assert lib.icv_ib_build(ctypes.byref(d), ctypes.byref(s), 1, 4, 0, L.ICV_I64, None, None) == L.ICV_ERR_ARG
    assert lib.icv_ib_build(ctypes.byref(d), ctypes.byref(s), 2, 4, 0, L.ICV_I64, None, None) == L.ICV_ERR_ARG
    assert lib.icv_ib_build(ctypes.byref(d), ctypes.byref(s), 1, 0, 0, L.ICV_I64, None, None) == L.ICV_ERR_ARG
    assert lib.icv_conv(ctypes.byref(d), ctypes.byref(s), 1, L.ICV_BF16, None, None, None, L.ICV_I64, 4, None,
                        None, None, None) == L.ICV_ERR_ARG
    assert "null" in L.last_error()
