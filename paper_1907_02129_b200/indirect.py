"""Indirect convolution on B200 — drop-in for the reference hot path
/root/reference/pkg/src/convbench/indirect.py.

Same names, signatures, argument meaning and error behaviour as the
reference (``ZERO_REF`` :36, ``make_zero_row`` :39-46, ``IndirectionBuffer``
:49-91, ``init_indirection_buffer`` :129-164, ``update_for_batch_growth``
:167-193, ``rebind_input`` :196-212, ``indirect_conv`` :239-300); the
difference is where the work runs.  Every buffer lives in HBM: the
indirection buffer is built by a device kernel (icv_ib_build) and the
convolution is an sm_100a indirect-GEMM kernel (icv_conv) that reads the
buffer's row references directly.  Nothing here computes on the CPU.

Buffer layout is the reference's: (T, R*S, mr) element offsets of the pixel
row each (output pixel, kernel tap) reads, ZERO_REF (-1) for padding taps,
tile-major then kernel element then lane (indirect.py:14-16), int64 by
default (``index_dtype=torch.int32`` halves its footprint).

``per_image=True`` stores only image 0's buffer, T = ceil(Ho*Wo/mr): the
canonical entry of image n is entry(0) + n*H*W*C (ZERO_REF kept), which the
kernels apply on the fly.  The reference leaves the row-reference
representation to the implementation; this form makes the
buffer independent of the batch (growth needs no rebuild) and small enough
to stay in L2 — for the 3-channel 7x7 stem the canonical buffer is 2.6x the
layer's compulsory HBM traffic.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib as L
from .errors import StaleBufferError
from .gemm import PackedFilter, TileConfig
from .tensors import ConvParams, NhwcTensor, Shape4, conv_output_shape

ZERO_REF = -1


def make_zero_row(channels: int, dtype: torch.dtype = torch.float32, device="cuda",
                  fill: int | float = 0) -> torch.Tensor:
    """The explicit zero vector substituted for out-of-bounds taps
    (indirect.py:39-46).  Shared read-only by buffers and operators.  For a
    uint8 convolution pass ``fill=input_zero_point`` so a padding tap means
    real 0."""
    if channels < 1:
        raise ValueError("channels must be >= 1")
    return torch.full((channels,), fill, dtype=dtype, device=device)


@dataclass(eq=False)
class IndirectionBuffer:
    """Ordered row references driving the indirect GEMM (indirect.py:49-91)."""

    mr: int
    batch: int
    out_h: int
    out_w: int
    params: ConvParams
    in_shape: Shape4
    input_data: torch.Tensor   # flat buffer of the bound input tensor
    zero_row: torch.Tensor
    offsets: torch.Tensor      # (tiles, R*S, mr) int64 (or int32), device resident
    per_image: bool = False    # offsets cover image 0 only (image-relative form)
    # offsets are exactly what icv_ib_build produced (always true for buffers
    # made by this module; an initialized buffer is immutable).
    # Lets channel-poor stride-2 layers read it at input-row granularity.
    canonical: bool = True
    # the zero row was all zero bytes when the buffer was initialized (it is
    # read-only by contract, indirect.py:42): stride-1 layers may then take
    # padding from TMA out-of-bounds zero fill (ICV_ZERO_ROW_ZEROS)
    zero_is_zero: bool = False
    # every byte of the zero row had this value at initialization (else None):
    # a uint8 zero row filled with the input zero point lets windowed layers
    # zero-fill padding and add a packed per-tap correction (ICV_ZERO_ROW_ZP)
    zero_fill_byte: "int | None" = None

    @property
    def pixel_count(self) -> int:
        return self.batch * self.out_h * self.out_w

    @property
    def tile_count(self) -> int:
        """Tiles of the canonical buffer this one represents."""
        return _tile_count(self.pixel_count, self.mr)

    @property
    def entry_count(self) -> int:
        """Entries of the canonical buffer (indirect.py:72-73)."""
        return self.tile_count * self.params.kernel_elems * self.mr

    @property
    def allocated_bytes(self) -> int:
        return self.offsets.numel() * self.offsets.element_size()

    def offsets_host(self) -> np.ndarray:
        """Host copy as the reference's canonical int64 (T, R*S, mr) buffer
        (a per-image buffer is expanded: entry(n) = entry(0) + n*H*W*C)."""
        offs = self.offsets.cpu().numpy().astype(np.int64)
        if not self.per_image:
            return offs
        ohw = self.out_h * self.out_w
        rs, mr = offs.shape[1], self.mr
        img = offs.transpose(0, 2, 1).reshape(-1, rs)[:ohw]             # (Ho*Wo, RS) per pixel of image 0
        p = np.minimum(np.arange(self.tile_count * mr), self.pixel_count - 1)
        n, q = p // ohw, p % ohw
        rows = img[q]
        step = self.in_shape.h * self.in_shape.w * self.in_shape.c
        rows = np.where(rows < 0, rows, rows + (n * step)[:, None])
        return rows.reshape(self.tile_count, mr, rs).transpose(0, 2, 1).copy()

    def verify(self) -> int:
        """Entries differing from the canonical buffer of this geometry
        (device check, icv_ib_check); a nonzero count clears `canonical` so
        the kernels gather tap by tap from whatever the buffer holds."""
        d, s = L.desc_of(self.params), L.shape_of(self.in_shape)
        fmt = L.TORCH_TO_ICV[self.offsets.dtype] | (L.ICV_IB_PER_IMAGE if self.per_image else 0)
        dev = self.offsets.device
        out = torch.zeros(1, dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            L.check(L.lib().icv_ib_check(ctypes.byref(d), ctypes.byref(s), self.batch, self.mr, fmt,
                                         L.ptr(self.offsets), L.ptr(out), L.stream_of(dev)), "icv_ib_check")
        bad = int(out.item())
        self.canonical = bad == 0
        return bad

    def rows_for_tile(self, t: int) -> list[torch.Tensor]:
        """Dereference tile t: R*S*mr pixel-row views in kernel-element order,
        mr rows per element; padding entries yield the zero row (:79-91)."""
        c = self.params.in_channels
        offs = self.offsets_host()[t].tolist()
        rows = []
        for e in range(self.params.kernel_elems):
            for m in range(self.mr):
                off = offs[e][m]
                rows.append(self.zero_row if off == ZERO_REF else self.input_data[off:off + c])
        return rows


def _tile_count(pixels: int, mr: int) -> int:
    return -(-pixels // mr)


def _build(in_shape: Shape4, params: ConvParams, batch: int, mr: int, offsets: torch.Tensor,
           first_tile: int, per_image: bool = False) -> None:
    d, s = L.desc_of(params), L.shape_of(in_shape)
    fmt = L.TORCH_TO_ICV[offsets.dtype] | (L.ICV_IB_PER_IMAGE if per_image else 0)
    with torch.cuda.device(offsets.device):
        L.check(L.lib().icv_ib_build(ctypes.byref(d), ctypes.byref(s), batch, mr, first_tile, fmt,
                                     L.ptr(offsets), L.stream_of(offsets.device)),
                "icv_ib_build")


def init_indirection_buffer(input: NhwcTensor, zero_row: torch.Tensor, params: ConvParams, out_shape: Shape4,
                            tile: TileConfig, batch: int | None = None, *,
                            index_dtype: torch.dtype = torch.int64, per_image: bool = False,
                            _zero_facts: tuple | None = None) -> IndirectionBuffer:
    """Build the buffer for ``input`` under ``params`` on the input's device
    (indirect.py:129-164).  ``batch`` limits initialization to the first
    images (extend later with update_for_batch_growth).  ``per_image=True``
    builds the batch-invariant image-relative form (module docstring)."""
    expected = conv_output_shape(params, input.shape)
    if out_shape != expected:
        raise ValueError(f"out_shape {out_shape} != computed {expected}")                 # :143-145
    if (not isinstance(zero_row, torch.Tensor) or zero_row.dtype != input.dtype
            or tuple(zero_row.shape) != (params.in_channels,)):
        raise ValueError(f"zero row must be {input.dtype} of length in_channels")         # :146-147
    batch = input.shape.n if batch is None else batch
    if not 1 <= batch <= input.shape.n:
        raise ValueError("batch must be within the physical input batch")                 # :148-150
    if index_dtype not in (torch.int64, torch.int32):
        raise ValueError("index_dtype must be torch.int64 or torch.int32")
    L.require_cuda(input.data, "input")
    if zero_row.device != input.data.device:
        raise ValueError("zero row must live on the input's device")
    pixels = (1 if per_image else batch) * out_shape.h * out_shape.w
    tiles = _tile_count(pixels, tile.mr)
    offsets = torch.empty((tiles, params.kernel_elems, tile.mr), dtype=index_dtype, device=input.data.device)
    _build(input.shape, params, batch, tile.mr, offsets, 0, per_image)
    if _zero_facts is None:
        # one scan of the (read-only, indirect.py:42) zero row: is it all zero
        # bytes, or one repeated byte (a uint8 zero point)?  (a host sync)
        zb = zero_row.reshape(-1).view(torch.uint8)
        lo, hi = (int(v) for v in torch.aminmax(zb))
        fill = lo if lo == hi else None
    else:   # facts of the same zero row, known from an earlier buffer
        fill = _zero_facts[1]
    return IndirectionBuffer(tile.mr, batch, out_shape.h, out_shape.w, params, input.shape, input.data,
                             zero_row, offsets, per_image, zero_is_zero=fill == 0, zero_fill_byte=fill)


def update_for_batch_growth(ib: IndirectionBuffer, new_batch: int) -> IndirectionBuffer:
    """Extend the buffer to more images of the same bound input
    (indirect.py:167-193): the old full-tile prefix is carried over verbatim
    (a device copy), only the old clamped boundary tile and the new region
    are built."""
    if new_batch < ib.batch:
        raise ValueError("cannot shrink a buffer; call indirect_conv with batch="
                         f"{new_batch} for logical truncation")
    if new_batch > ib.in_shape.n:
        raise ValueError("new batch exceeds the bound input tensor's batch")
    if new_batch == ib.batch:
        return ib
    if ib.per_image:                       # image-relative entries serve every image: nothing to build
        return replace(ib, batch=new_batch)
    keep = ib.pixel_count // ib.mr                                                        # :185
    tiles = _tile_count(new_batch * ib.out_h * ib.out_w, ib.mr)
    offsets = torch.empty((tiles, ib.params.kernel_elems, ib.mr), dtype=ib.offsets.dtype, device=ib.offsets.device)
    if keep:
        offsets[:keep].copy_(ib.offsets[:keep])                                           # :188
    _build(ib.in_shape, ib.params, new_batch, ib.mr, offsets, keep)                       # :189-192
    return replace(ib, batch=new_batch, offsets=offsets)


def rebind_input(ib: IndirectionBuffer, new_input: NhwcTensor, new_zero: torch.Tensor) -> IndirectionBuffer:
    """Complete reinitialization against a new input tensor and zero row
    (indirect.py:196-212).  The new input must have the buffer's shape."""
    if new_input.shape != ib.in_shape:
        raise ValueError(f"rebind requires identical shape; buffer has {ib.in_shape}, "
                         f"new input has {new_input.shape}")
    out_shape = Shape4(new_input.shape.n, ib.out_h, ib.out_w, ib.params.out_channels)
    facts = (ib.zero_is_zero, ib.zero_fill_byte) if new_zero is ib.zero_row else None
    return init_indirection_buffer(new_input, new_zero, ib.params, out_shape, TileConfig(mr=ib.mr),
                                   batch=ib.batch, index_dtype=ib.offsets.dtype, per_image=ib.per_image,
                                   _zero_facts=facts)


def indirect_gemm_microkernel(kernel_elems: int, channels: int, packed_b_tile: torch.Tensor,
                              row_refs: list[torch.Tensor], acc: torch.Tensor) -> torch.Tensor:
    """Single-tile semantics of the indirect GEMM (indirect.py:215-236; the
    paper's Listing 3): per kernel element load ``mr`` fresh row references
    and accumulate ``channels``-long dot products into ``acc`` (mr, nr), in
    kernel-element-major, channel-minor order with one rounded multiply and
    one rounded add per product (gemm.py:6-15) -- bit-exact with the
    reference for float32.  Element-wise torch ops on whatever device the
    tensors live on; it defines what one tile of ``icv_conv`` computes (the
    tests compare the two) and is not itself the hot path.
    ``packed_b_tile`` is ``PackedFilter.tile(jt)``; ``row_refs`` is
    ``IndirectionBuffer.rows_for_tile(t)``."""
    mr = acc.shape[0]
    if len(row_refs) < kernel_elems * mr:
        raise ValueError("row_refs must hold kernel_elems * mr rows")
    k = 0
    for e in range(kernel_elems):
        rows = torch.stack([r[:channels] for r in row_refs[e * mr:(e + 1) * mr]]).to(acc.dtype)   # (mr, C)
        for c in range(channels):
            acc += rows[:, c:c + 1] * packed_b_tile[k].to(acc.dtype)
            k += 1
    return acc


def _check_filter(pf: PackedFilter, params: ConvParams) -> None:
    # im2col.py:150-156
    if (pf.kernel_elems != params.kernel_elems or pf.in_channels != params.in_channels
            or pf.k_out != params.out_channels):
        raise ValueError("packed filter does not match convolution params")


def _same_binding(bound: torch.Tensor, data: torch.Tensor) -> bool:
    """The reference checks array identity (indirect.py:254).  On the device
    the binding is the buffer itself: same tensor object, or the same
    device allocation viewed with the same dtype and extent."""
    if bound is data:
        return True
    return (bound.device == data.device and bound.dtype == data.dtype and bound.numel() == data.numel()
            and bound.data_ptr() == data.data_ptr())


ALGORITHMS = ("auto", "gather")


def conv_flags(ib: IndirectionBuffer, pf: PackedFilter, dtype: torch.dtype, algorithm: str = "auto") -> int:
    """The ``ib_dtype`` argument of icv_conv: index type plus the layout
    facts the host knows about this buffer and zero row."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"algorithm must be one of {ALGORITHMS}")
    return (L.TORCH_TO_ICV[ib.offsets.dtype] | (L.ICV_IB_PER_IMAGE if ib.per_image else 0)
            | (L.ICV_IB_CANONICAL if ib.canonical else 0)
            | (L.ICV_ZERO_ROW_ZEROS if ib.zero_is_zero else 0)
            | (L.ICV_ZERO_ROW_ZP if (dtype == torch.uint8 and pf.quant is not None
                                     and ib.zero_fill_byte == pf.quant.input_zero_point) else 0)
            | (L.ICV_PREFER_GATHER if algorithm == "gather" else 0))


def indirect_conv(input: NhwcTensor, pf: PackedFilter, ib: IndirectionBuffer, params: ConvParams,
                  tile: TileConfig, batch: int | None = None, *, out: NhwcTensor | None = None,
                  algorithm: str = "auto") -> NhwcTensor:
    """Convolution through the indirection buffer; no patch matrix exists
    (indirect.py:239-300).  ``batch`` may name fewer images than the buffer
    covers (logical truncation); anything else the buffer was not built for
    raises StaleBufferError.  Output dtype: float32 for float32 input
    (bit-exact with the reference), bfloat16 for bfloat16, uint8 for uint8.
    ``out`` optionally supplies a preallocated output tensor.

    ``algorithm="gather"`` runs the IB-gather kernels (every A row fetched
    through its buffer entry, the paper's Listing 3 mainloop) instead of the
    specialisations a canonical buffer permits (sliding windows for
    stride-1 R*S > 1 layers, row-sliding for the channel-poor stem, dense
    TMA rows for 1x1 layers); the results agree within the dtype's contract
    (bit-exact for uint8 and float32)."""
    _check_filter(pf, params)                                                             # :253
    if not _same_binding(ib.input_data, input.data):
        raise StaleBufferError("buffer is bound to a different input tensor; rebind_input first")   # :254-257
    if ib.params != params:
        raise StaleBufferError("buffer was built for different conv params")            # :258-259
    if ib.in_shape != input.shape:
        raise StaleBufferError("input shape changed; rebuild the buffer")               # :260-261
    if ib.mr != tile.mr or pf.nr != tile.nr:
        raise StaleBufferError("tile configuration differs from buffer/packing")        # :262-263
    batch = ib.batch if batch is None else batch
    if not 1 <= batch <= ib.batch:
        raise ValueError("batch must be <= the initialized buffer batch; use "
                         "update_for_batch_growth to extend it")                          # :265-270
    if input.dtype != pf.dtype:
        raise ValueError(f"input dtype {input.dtype} does not match the packed filter's compute dtype {pf.dtype}")
    if ib.zero_row.dtype != input.dtype:
        raise ValueError("zero row dtype does not match the input")
    L.require_cuda(input.data, "input")
    dev = input.data.device
    if pf.packed.device != dev or ib.offsets.device != dev or ib.zero_row.device != dev:
        raise ValueError("input, packed filter, indirection buffer and zero row must share one device")
    out_shape = Shape4(batch, ib.out_h, ib.out_w, pf.k_out)
    if out is None:
        out = NhwcTensor.empty(out_shape, dtype=input.dtype, device=dev)
    elif out.shape != out_shape or out.dtype != input.dtype or out.data.device != dev:
        raise ValueError(f"out must be a {input.dtype} NhwcTensor of shape {out_shape} on {dev}")
    d, s = L.desc_of(params), L.shape_of(input.shape)
    q = L.quant_of(pf.quant)
    flags = conv_flags(ib, pf, input.dtype, algorithm)
    with torch.cuda.device(dev):
        L.check(L.lib().icv_conv(ctypes.byref(d), ctypes.byref(s), batch, L.TORCH_TO_ICV[input.dtype],
                                 L.ptr(input.data), L.ptr(ib.zero_row), L.ptr(ib.offsets), flags,
                                 ib.mr, L.ptr(pf.packed),
                                 ctypes.byref(q) if q is not None else None, L.ptr(out.data), L.stream_of(dev)),
                "icv_conv")
    return out
