"""Oracle: float convolution through the indirection buffer (TEST INFRASTRUCTURE ONLY).

Restates the reference's arithmetic contract (gemm.py:6-15, reference.py:1-12):
each output accumulates, starting from its bias (or +0.0), one product per
(kernel element e ascending, channel c ascending), the product and the sum
each rounded separately to float32 (no FMA).  ``indirect_conv_f32`` follows
indirect.py:272-300 exactly (per-tap gather with padding rows replaced by the
zero row, then C multiply/add passes); the mr x nr register tiling of the
reference does not change any per-element operation sequence, so it is not
reproduced.  ``direct_conv_f32`` restates reference.py:30-84 (skips padding
taps) and is the second, independent oracle.

bf16 (BASELINE cfg2/3): inputs and weights are rounded to bf16 with
round-to-nearest-even (``bf16_round``), then the f32 oracle runs on those
values.
"""

from __future__ import annotations

import numpy as np

from .ib import ZERO_REF, out_hw


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even) and return
    them widened back to float32.  NaN stays NaN."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(a)
    out = r.astype(np.uint32).view(np.float32).copy()
    out[nan] = np.float32("nan")
    return out


def pixel_refs(offsets: np.ndarray, pixels: int, pixel_index: np.ndarray | None = None) -> np.ndarray:
    """(P_sel, RS) row references of the selected output pixels, read from a
    (T, RS, mr) buffer at ((p // mr)*RS + e)*mr + p % mr (indirect.py:14-16)."""
    t, rs, mr = offsets.shape
    p = np.arange(pixels, dtype=np.int64) if pixel_index is None else np.asarray(pixel_index, np.int64)
    return offsets[p // mr, :, p % mr]


def indirect_conv_f32(x_flat: np.ndarray, zero_row: np.ndarray, offsets: np.ndarray,
                      params, w_krsc: np.ndarray, bias: np.ndarray | None,
                      batch: int, out_h: int, out_w: int,
                      pixel_index: np.ndarray | None = None) -> np.ndarray:
    """(pixels, K) float32 output (or the ``pixel_index`` rows of it);
    indirect.py:272-300.

    ``offsets`` is the (T, RS, mr) int64 buffer.  The reference computes the
    clamped tail lanes and drops them (:296-300); rows are independent, so
    only the real (or selected) pixels are computed here.
    """
    c = params.in_channels
    k = params.out_channels
    rs = params.kernel_h * params.kernel_w
    refs = pixel_refs(offsets, batch * out_h * out_w, pixel_index)
    w = np.ascontiguousarray(w_krsc, dtype=np.float32).reshape(k, rs, c)
    acc = np.empty((refs.shape[0], k), dtype=np.float32)
    acc[:] = np.zeros(k, np.float32) if bias is None else np.asarray(bias, np.float32)
    tmp = np.empty_like(acc)
    ch = np.arange(c, dtype=np.int64)
    for e in range(rs):
        off = refs[:, e]
        rows = np.take(x_flat, np.maximum(off, 0)[:, None] + ch)
        rows[off == ZERO_REF] = zero_row
        we = w[:, e, :]
        for ic in range(c):
            np.multiply(rows[:, ic, None], we[None, :, ic], out=tmp)
            np.add(acc, tmp, out=acc)
    return acc


def direct_conv_f32(x4: np.ndarray, w_krsc: np.ndarray, bias: np.ndarray | None,
                    params) -> np.ndarray:
    """(n, out_h, out_w, K) float32; reference.py:30-84 (padding taps
    skipped, ky -> kx -> ic order, bias as accumulator init)."""
    n, h, w_in, c = x4.shape
    oh, ow = out_hw(params, h, w_in)
    k = params.out_channels
    w4 = np.ascontiguousarray(w_krsc, np.float32).reshape(k, params.kernel_h, params.kernel_w, c)
    out = np.zeros((n, oh, ow, k), np.float32)
    if bias is not None:
        out[...] = bias
    tmp = np.empty((n, oh, ow, k), np.float32)
    oy = np.arange(oh)
    ox = np.arange(ow)
    for ky in range(params.kernel_h):
        iy = oy * params.stride_h + ky * params.dilation_h - params.pad_top
        vy = (iy >= 0) & (iy < h)
        for kx in range(params.kernel_w):
            ix = ox * params.stride_w + kx * params.dilation_w - params.pad_left
            vx = (ix >= 0) & (ix < w_in)
            if not vy.any() or not vx.any():
                continue
            yi, xi = np.nonzero(vy)[0], np.nonzero(vx)[0]
            taps = x4[:, iy[yi]][:, :, ix[xi]]  # (n, |yi|, |xi|, c)
            dst = out[:, yi[0]:yi[-1] + 1, xi[0]:xi[-1] + 1, :]
            t = tmp[:, :len(yi), :len(xi), :]
            for ic in range(c):
                np.multiply(taps[..., ic:ic + 1], w4[:, ky, kx, ic], out=t)
                np.add(dst, t, out=dst)
    return out
