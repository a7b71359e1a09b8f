"""Oracle: indirection-buffer construction (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/convbench/indirect.py:94-126 (tile count and
``_compute_offsets``), :185-192 (batch growth) and tensors.py:184-211
(output shape).  ``params`` is any object exposing the ConvParams field names
(kernel_h, kernel_w, stride_h, stride_w, dilation_h, dilation_w, pad_top,
pad_left, pad_bottom, pad_right, in_channels, out_channels); shapes are
(n, h, w, c) tuples.
"""

from __future__ import annotations

import numpy as np

ZERO_REF = -1  # indirect.py:36


def out_hw(params, in_h: int, in_w: int) -> tuple[int, int]:
    """Output extent; tensors.py:195-211.  Returns (0, 0) if the dilated
    kernel does not fit (the reference raises InvalidGeometryError)."""
    span_h = in_h + params.pad_top + params.pad_bottom - params.dilation_h * (params.kernel_h - 1) - 1
    span_w = in_w + params.pad_left + params.pad_right - params.dilation_w * (params.kernel_w - 1) - 1
    if span_h < 0 or span_w < 0:
        return 0, 0
    return span_h // params.stride_h + 1, span_w // params.stride_w + 1


def tile_count(pixels: int, mr: int) -> int:
    """ceil(pixels / mr); indirect.py:94-95."""
    return -(-pixels // mr)


def compute_offsets(in_shape, params, out_h: int, out_w: int, batch: int, mr: int,
                    first_tile: int = 0) -> np.ndarray:
    """Offsets for tiles [first_tile, T) as int64 (T - first_tile, R*S, mr).

    indirect.py:98-126: lane = t*mr + m, clamped to the last real pixel
    (:111); (n, oy, ox) decomposition (:112-114); per tap
    iy = oy*SY + ky*DY - PT, ix = ox*SX + kx*DX - PL (:120-121); valid taps
    store the element offset ((n*H + iy)*W + ix)*C of the pixel row, padding
    taps store ZERO_REF (:122-125).
    """
    _, h, w, c = in_shape
    pixels = batch * out_h * out_w
    tiles = tile_count(pixels, mr)
    lane = np.arange(first_tile * mr, tiles * mr, dtype=np.int64)
    p = np.minimum(lane, pixels - 1)
    n = p // (out_h * out_w)
    oy = (p // out_w) % out_h
    ox = p % out_w
    rs = params.kernel_h * params.kernel_w
    out = np.empty((tiles - first_tile, rs, mr), dtype=np.int64)
    for ky in range(params.kernel_h):
        iy = oy * params.stride_h + ky * params.dilation_h - params.pad_top
        for kx in range(params.kernel_w):
            ix = ox * params.stride_w + kx * params.dilation_w - params.pad_left
            valid = (iy >= 0) & (iy < h) & (ix >= 0) & (ix < w)
            off = ((n * h + iy) * w + ix) * c
            out[:, ky * params.kernel_w + kx, :] = np.where(valid, off, ZERO_REF).reshape(-1, mr)
    return out


def grow_offsets(old: np.ndarray, in_shape, params, out_h: int, out_w: int,
                 old_batch: int, new_batch: int, mr: int) -> np.ndarray:
    """update_for_batch_growth, indirect.py:185-192: keep the old full-tile
    prefix verbatim, recompute the clamped boundary tile and the new region."""
    keep = (old_batch * out_h * out_w) // mr
    tiles = tile_count(new_batch * out_h * out_w, mr)
    rs = params.kernel_h * params.kernel_w
    out = np.empty((tiles, rs, mr), dtype=np.int64)
    out[:keep] = old[:keep]
    out[keep:] = compute_offsets(in_shape, params, out_h, out_w, new_batch, mr, first_tile=keep)
    return out


def entry_offset(p: int, e: int, mr: int, rs: int) -> int:
    """Flat position of (pixel p, tap e) in a (T, RS, mr) buffer: the layout
    is tile-major, then kernel element, then lane (indirect.py:14-16)."""
    return ((p // mr) * rs + e) * mr + p % mr
