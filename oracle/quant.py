"""Oracle: QNNPACK-style asymmetric uint8 convolution (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED AGAINST THE REFERENCE: the reference is float32-only
(tensors.py:107-108; quantized kernels are out of scope), so
there is no reference output to pin this against.  It follows the
reference's indirection buffer (indirect.py:98-126) and loop order
(indirect.py:287-294) with the integer semantics fixed in SURVEY.md
Appendix A.3, and is pinned by this repo's own known-answer tests
(tests/test_oracle_quant.py).

Semantics:
  zero row   = C bytes equal to the input zero point, so padding taps
               contribute (zx - zx) * (w - zw) = 0;
  acc[p, k]  = bias[k] + sum_{e, c} (x - zx) * (w - zw)   (exact, int32 range);
  requant    = gemmlowp/QNNPACK "q31": y = SRDHM(acc, M0);
               y = RoundingDivideByPOT(y, shift) (half away from zero);
               y += zo; clamp to [qmin, qmax].
  multiplier = real = (f64(sx) * f64(sw)) / f64(so);  real = q * 2**e with
               q in [0.5, 1);  M0 = round_half_away(q * 2**31);
               if M0 == 2**31: M0 = 2**30, e += 1;  shift = -e.
"""

from __future__ import annotations

import math

import numpy as np

from .ib import ZERO_REF

INT32_MIN = -(1 << 31)
INT32_MAX = (1 << 31) - 1


def requant_params(input_scale: float, kernel_scale: float, output_scale: float) -> tuple[int, int]:
    """(M0, shift) for real_scale = sx*sw/so computed in float64 from the
    float32 scales."""
    sx = float(np.float32(input_scale))
    sw = float(np.float32(kernel_scale))
    so = float(np.float32(output_scale))
    real = (sx * sw) / so
    if not (0.0 < real < 1.0):
        raise ValueError(f"requantization scale {real} must be in (0, 1)")
    q, e = math.frexp(real)
    m0 = int(math.floor(q * (1 << 31) + 0.5))
    if m0 == (1 << 31):
        m0 = 1 << 30
        e += 1
    shift = -e
    if not 0 <= shift <= 31:
        raise ValueError(f"requantization shift {shift} out of [0, 31]")
    return m0, shift


def srdhm(a: np.ndarray, b: int) -> np.ndarray:
    """SaturatingRoundingDoublingHighMul on int32 values held in int64."""
    a = np.asarray(a, dtype=np.int64)
    ab = a * np.int64(b)
    nudge = np.where(ab >= 0, np.int64(1 << 30), np.int64(1 - (1 << 30)))
    s = ab + nudge
    # C integer division by 2**31 truncates toward zero
    q = np.where(s >= 0, s >> 31, -((-s) >> 31))
    sat = (a == INT32_MIN) & (b == INT32_MIN)
    return np.where(sat, np.int64(INT32_MAX), q)


def rounding_divide_by_pot(x: np.ndarray, exponent: int) -> np.ndarray:
    """gemmlowp RoundingDivideByPOT: arithmetic shift, ties away from zero."""
    x = np.asarray(x, dtype=np.int64)
    mask = np.int64((1 << exponent) - 1)
    remainder = x & mask
    threshold = (mask >> 1) + np.where(x < 0, np.int64(1), np.int64(0))
    return (x >> exponent) + np.where(remainder > threshold, np.int64(1), np.int64(0))


def requantize(acc: np.ndarray, m0: int, shift: int, out_zp: int,
               qmin: int = 0, qmax: int = 255) -> np.ndarray:
    y = rounding_divide_by_pot(srdhm(acc, m0), shift) + out_zp
    return np.clip(y, qmin, qmax).astype(np.uint8)


def indirect_conv_acc(x_flat: np.ndarray, zero_row: np.ndarray, offsets: np.ndarray,
                      params, w_krsc: np.ndarray, bias: np.ndarray | None,
                      batch: int, out_h: int, out_w: int,
                      input_zp: int, kernel_zp: int,
                      pixel_index: np.ndarray | None = None) -> np.ndarray:
    """int64 (pixels, K) accumulators: bias + sum (x - zx)(w - zw), walking the
    buffer per tap as indirect.py:287-294 does (integer sums are exact, so the
    order is immaterial).  ``pixel_index`` selects a subset of output rows."""
    from .conv import pixel_refs

    c = params.in_channels
    k = params.out_channels
    rs = params.kernel_h * params.kernel_w
    refs = pixel_refs(offsets, batch * out_h * out_w, pixel_index)
    w = np.asarray(w_krsc).reshape(k, rs, c).astype(np.int64) - kernel_zp
    acc = np.zeros((refs.shape[0], k), dtype=np.int64)
    if bias is not None:
        acc[:] = np.asarray(bias, dtype=np.int64)
    ch = np.arange(c, dtype=np.int64)
    for e in range(rs):
        off = refs[:, e]
        rows = np.take(x_flat, np.maximum(off, 0)[:, None] + ch).astype(np.int64)
        rows[off == ZERO_REF] = np.asarray(zero_row, dtype=np.int64)
        # exact int64 contraction (no float rounding anywhere)
        acc += np.einsum("pc,kc->pk", rows - input_zp, w[:, e, :], dtype=np.int64)
    return acc


def indirect_conv_u8(x_flat, zero_row, offsets, params, w_krsc, bias, batch, out_h, out_w,
                     input_zp, input_scale, kernel_zp, kernel_scale, output_zp, output_scale,
                     qmin: int = 0, qmax: int = 255,
                     pixel_index: np.ndarray | None = None) -> np.ndarray:
    """uint8 (pixels, K) output of the quantized indirect convolution."""
    acc = indirect_conv_acc(x_flat, zero_row, offsets, params, w_krsc, bias, batch,
                            out_h, out_w, input_zp, kernel_zp, pixel_index)
    if acc.min(initial=0) < INT32_MIN or acc.max(initial=0) > INT32_MAX:
        raise OverflowError("int32 accumulator overflow")
    m0, shift = requant_params(input_scale, kernel_scale, output_scale)
    return requantize(acc, m0, shift, output_zp, qmin, qmax)
