"""Direct convolution on the device -- the correctness oracle of the GPU
benchmark harness; drop-in for convbench.reference.direct_conv
(/root/reference/pkg/src/convbench/reference.py:30-84).

Same contract: bias as the accumulator's initial value, then kernel row,
kernel column, input channel ascending, one rounded multiply and one
rounded add per tap (no FMA), padding taps skipped.  It runs as its own
kernel (``icv_direct_conv``, csrc/direct_conv.cu) that never touches an
indirection buffer, so it checks the indirect path independently.  float32
inputs give float32 outputs bit-exact with the reference; bfloat16 inputs
are widened exactly, so the result is the reference's float32 convolution
of the bf16 operands (the bf16 tolerance oracle of SURVEY.md Appendix A.2).
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib as L
from .tensors import ConvParams, FilterTensor, NhwcTensor, conv_output_shape


def direct_conv(input: NhwcTensor, filt: FilterTensor, bias, params: ConvParams) -> NhwcTensor:
    """Convolve ``input`` with ``filt`` (reference.py:30-84); a fresh float32
    NHWC output.  ValueError on channel/filter mismatches; InvalidGeometryError
    for degenerate geometry (from conv_output_shape)."""
    if not filt.matches(params):
        raise ValueError("filter dimensions do not match params")
    out_shape = conv_output_shape(params, input.shape)
    if input.dtype not in (torch.float32, torch.bfloat16) or filt.dtype not in (torch.float32, torch.bfloat16):
        raise TypeError("direct_conv takes float32 or bfloat16 tensors")
    L.require_cuda(input.data, "input")
    dev = input.data.device
    w = filt.data.to(dev)
    b = None
    if bias is not None:
        b = torch.as_tensor(bias)
        if b.dtype != torch.float32 or tuple(b.shape) != (params.out_channels,):
            raise ValueError("bias must be float32 of length out_channels")
        b = b.to(dev)
    out = NhwcTensor.empty(out_shape, dtype=torch.float32, device=dev)
    d, s = L.desc_of(params), L.shape_of(input.shape)
    with torch.cuda.device(dev):
        L.check(L.lib().icv_direct_conv(ctypes.byref(d), ctypes.byref(s), input.shape.n,
                                        L.TORCH_TO_ICV[input.dtype], L.ptr(input.data), L.TORCH_TO_ICV[w.dtype],
                                        L.ptr(w), L.ptr(b) if b is not None else None, L.ptr(out.data),
                                        L.stream_of(dev)), "icv_direct_conv")
    return out
