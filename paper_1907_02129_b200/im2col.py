"""GEMM-based convolution on the device: the baseline the indirect algorithm
is measured against (reference im2col.py; §2.1 / Figure 1).

``build_patch_matrix`` materializes the im2row matrix with ``icv_im2col``
(an HBM-bound copy, R*S times the input); ``gemm_conv`` / ``gemm_only``
multiply it with the filter on the same tcgen05 kernels as the indirect
path, by running the product as a 1x1 convolution over the patch matrix
(one image of 1 x P pixels with R*S*C channels: the packed filter of that
view holds the same KRSC bytes).  So the two variants differ exactly by the
patch matrix, which is the paper's comparison.  Float32 is bit-exact with
the reference's gemm_conv (same bias init and ascending-k order,
im2col.py:117-131 / gemm.py:6-15); bf16 and uint8 match indirect_conv.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib as L
from .gemm import PackedFilter, TileConfig, pack_filter
from .indirect import _check_filter, indirect_conv, init_indirection_buffer, make_zero_row
from .tensors import ConvParams, FilterTensor, NhwcTensor, Shape4, conv_output_shape


@dataclass(eq=False)
class PatchMatrix:
    """The materialized im2row buffer plus bookkeeping (im2col.py:21-45).

    ``allocated_bytes`` is 0 when ``matrix`` is a view of the input
    (pointwise unit-stride fast path, im2col.py:69-73)."""

    matrix: torch.Tensor          # (rows, cols) on the input's device
    params: ConvParams
    input_shape: Shape4
    out_shape: Shape4
    is_view: bool
    _gemm: dict = field(default_factory=dict, repr=False)   # cached 1x1-view buffer for gemm_only

    @property
    def rows(self) -> int:
        return self.matrix.shape[0]

    @property
    def cols(self) -> int:
        return self.matrix.shape[1]

    @property
    def allocated_bytes(self) -> int:
        return 0 if self.is_view else self.matrix.numel() * self.matrix.element_size()


def build_patch_matrix(input: NhwcTensor, params: ConvParams, out: PatchMatrix | None = None, *,
                       zero_row: torch.Tensor | None = None) -> PatchMatrix:
    """Gather every output pixel's taps into one matrix row (im2col.py:48-114):
    row p, column e*C + c = input at (oy*SY + ky*DY - PT, ox*SX + kx*DX - PL),
    or the padding value (zeros, or ``zero_row`` -- uint8: the zero point).
    ``out`` refills a previously built matrix of the same geometry."""
    if input.shape.c != params.in_channels:
        raise ValueError("input channel count does not match params")                 # :66-67
    out_shape = conv_output_shape(params, input.shape)
    m = out_shape.n * out_shape.h * out_shape.w
    cols = params.kernel_elems * params.in_channels
    L.require_cuda(input.data, "input")
    if params.is_pointwise_unit_stride():                                                # :69-73
        return PatchMatrix(input.data.view(m, cols), params, input.shape, out_shape, is_view=True)
    dev = input.data.device
    if out is None:
        matrix = torch.empty((m, cols), dtype=input.dtype, device=dev)
    else:
        if out.is_view or out.params != params or out.input_shape != input.shape:
            raise ValueError("provided patch matrix was built for other geometry")      # :80-82
        matrix = out.matrix
        # (the reference is float32-only; with several dtypes the buffer's
        # element type, device and extent must match too, or the kernel
        # would write past it)
        if matrix.dtype != input.dtype or matrix.device != dev or matrix.numel() != m * cols:
            raise ValueError(f"provided patch matrix is {matrix.dtype} x {matrix.numel()} on {matrix.device}; "
                             f"this input needs {input.dtype} x {m * cols} on {dev}")
    if zero_row is not None and (zero_row.numel() != params.in_channels or zero_row.dtype != input.dtype
                                 or zero_row.device != dev):
        raise ValueError("zero_row must hold in_channels elements of the input dtype on its device")
    d, s = L.desc_of(params), L.shape_of(input.shape)
    with torch.cuda.device(dev):
        L.check(L.lib().icv_im2col(ctypes.byref(d), ctypes.byref(s), input.shape.n, L.TORCH_TO_ICV[input.dtype],
                                   L.ptr(input.data), L.ptr(zero_row) if zero_row is not None else None,
                                   L.ptr(matrix), L.stream_of(dev)),
                "icv_im2col")
    if out is not None:
        return out
    return PatchMatrix(matrix, params, input.shape, out_shape, is_view=False)


def _gemm_view(pf: PackedFilter, tile: TileConfig) -> PackedFilter:
    """The packed filter of the 1x1 view (K x 1 x 1 x R*S*C, same bytes)."""
    view = getattr(pf, "_gemm_view", None)
    if view is not None and view.nr == tile.nr:
        return view
    red = pf.kernel_elems * pf.in_channels
    p1 = ConvParams(1, 1, in_channels=red, out_channels=pf.k_out)
    filt = FilterTensor(pf.k_out, 1, 1, red, pf.krsc)
    view = pack_filter(filt, pf.bias, p1, tile, compute_dtype=pf.dtype, quant=pf.quant)
    pf._gemm_view = view
    return view


def gemm_only(prebuilt: PatchMatrix, pf: PackedFilter, tile: TileConfig) -> torch.Tensor:
    """The matrix multiply alone over an already-built patch matrix
    (im2col.py:134-147); returns the (rows, K) output matrix."""
    _check_filter(pf, prebuilt.params)
    if prebuilt.cols != pf.reduction_len:
        raise ValueError("patch matrix columns do not match packed filter")             # :144-145
    view = _gemm_view(pf, tile)
    m = prebuilt.matrix
    key = (m.data_ptr(), prebuilt.rows, prebuilt.cols, m.dtype, m.device, tile.mr, tile.nr)
    # the buffer of the 1 x P view is built once per patch-matrix location;
    # a pointwise layer's "patch matrix" is a fresh view of the input each
    # call, so its buffer is cached on the packed filter, keyed by location
    store = prebuilt._gemm if not prebuilt.is_view else pf.__dict__.setdefault("_gemm_ib_cache", {})
    cached = store.get("ib") if not prebuilt.is_view else store.get(key)
    if cached is None or cached[0] != key:
        x1 = NhwcTensor(Shape4(1, 1, prebuilt.rows, prebuilt.cols), m.view(-1))
        fill = pf.quant.input_zero_point if pf.quant is not None else 0
        zero = make_zero_row(prebuilt.cols, dtype=m.dtype, device=m.device, fill=fill)
        ib = init_indirection_buffer(x1, zero, view.params, conv_output_shape(view.params, x1.shape), tile)
        cached = (key, x1, ib)
        if prebuilt.is_view:
            if len(store) >= 8:
                store.clear()
            store[key] = cached
        else:
            store["ib"] = cached
    _, x1, ib = cached
    y = indirect_conv(x1, view, ib, view.params, tile)
    return y.data.view(prebuilt.rows, pf.k_out)


def gemm_conv(input: NhwcTensor, pf: PackedFilter, params: ConvParams, tile: TileConfig,
              patch: PatchMatrix | None = None) -> NhwcTensor:
    """im2row followed by the GEMM (im2col.py:117-131); a fresh NHWC output.
    uint8 padding taps take the input zero point (the quantized zero row)."""
    _check_filter(pf, params)
    zero = None
    if input.dtype == torch.uint8 and pf.quant is not None:
        zero = make_zero_row(params.in_channels, dtype=torch.uint8, device=input.data.device,
                             fill=pf.quant.input_zero_point)
    pm = build_patch_matrix(input, params, out=patch, zero_row=zero)
    y = gemm_only(pm, pf, tile)
    return NhwcTensor(pm.out_shape, y.reshape(-1))
