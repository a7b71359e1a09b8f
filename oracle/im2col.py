"""Oracle: im2row patch matrix (TEST INFRASTRUCTURE ONLY).

Restates the reference's build_patch_matrix (im2col.py:48-114) in numpy:
row p = output pixel (n, oy, ox row-major), column e*C + c with
e = ky*S + kx holds the input at iy = oy*SY + ky*DY - PT,
ix = ox*SX + kx*DX - PL, or ``pad`` (the reference's 0.0) out of bounds.
Pinned against the reference's own outputs by tests/golden/im2col_golden.json
(oracle/gen_golden_im2col.py).  Only tests/ use it, as the checker.
"""

from __future__ import annotations

import numpy as np


def out_hw(p, h: int, w: int) -> tuple[int, int]:
    """conv_output_shape (tensors.py:184-211)."""
    oh = (h + p.pad_top + p.pad_bottom - p.dilation_h * (p.kernel_h - 1) - 1) // p.stride_h + 1
    ow = (w + p.pad_left + p.pad_right - p.dilation_w * (p.kernel_w - 1) - 1) // p.stride_w + 1
    return oh, ow


def patch_matrix(x: np.ndarray, p, n: int, h: int, w: int, pad=None) -> np.ndarray:
    """x: flat NHWC (n, h, w, C); returns (n*oh*ow, R*S*C)."""
    c = p.in_channels
    oh, ow = out_hw(p, h, w)
    x4 = x.reshape(n, h, w, c)
    out = np.zeros((n, oh, ow, p.kernel_h * p.kernel_w, c), dtype=x.dtype)
    if pad is not None:
        out[...] = np.asarray(pad, dtype=x.dtype).reshape(c)
    for ky in range(p.kernel_h):                                                      # im2col.py:90-113
        for kx in range(p.kernel_w):
            e = ky * p.kernel_w + kx
            for oy in range(oh):
                iy = oy * p.stride_h + ky * p.dilation_h - p.pad_top
                if not 0 <= iy < h:
                    continue
                for ox in range(ow):
                    ix = ox * p.stride_w + kx * p.dilation_w - p.pad_left
                    if 0 <= ix < w:
                        out[:, oy, ox, e, :] = x4[:, iy, ix, :]
    return out.reshape(n * oh * ow, p.kernel_h * p.kernel_w * c)


def gemm_conv_f32(mat: np.ndarray, wk: np.ndarray, bias: np.ndarray) -> np.ndarray:
    """out[p, k] = bias[k] (+) sum_j mat[p, j] (x) w[k, j], ascending j, separate
    float32 multiply and add (gemm.py:6-15)."""
    k_out = bias.shape[0]
    w2 = wk.reshape(k_out, -1).astype(np.float32)
    acc = np.broadcast_to(bias.astype(np.float32), (mat.shape[0], k_out)).copy()
    for j in range(mat.shape[1]):
        acc = np.add(acc, np.multiply(mat[:, j:j + 1], w2[:, j][None, :], dtype=np.float32), dtype=np.float32)
    return acc
