"""Tile configuration and filter packing — drop-in for the hot-path part of
/root/reference/pkg/src/convbench/gemm.py (``TileConfig`` :37-46,
``PackedFilter`` :94-132, ``pack_filter`` :135-167).

On the GPU the weights are repacked once, on the device, into the layout the
selected kernel reads (K-major 128-byte column blocks for the tcgen05
kernels; KRSC for the exact-f32 and CUDA-core kernels), and the bias — plus,
for uint8, the zero-point corrections — is folded into one epilogue constant
per output channel.  ``nr`` stays the reference's API tag: it must match the
``TileConfig`` passed to ``indirect_conv`` (indirect.py:262-263) but the
device tile width is chosen by the kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .tensors import ConvParams, FilterTensor


@dataclass(frozen=True)
class TileConfig:
    """mr = indirection-buffer tile height (rows of the (T, R*S, mr) layout);
    nr = packing tag (gemm.py:37-46)."""

    mr: int = 4
    nr: int = 8

    def __post_init__(self):
        if self.mr < 1 or self.nr < 1:
            raise ValueError("tile dimensions must be >= 1")


@dataclass(frozen=True)
class QuantParams:
    """Asymmetric uint8 quantization of one convolution (QNNPACK style).
    No reference counterpart: the reference is float32-only (tensors.py:107-108)."""

    input_zero_point: int
    input_scale: float
    kernel_zero_point: int
    kernel_scale: float
    output_zero_point: int
    output_scale: float
    output_min: int = 0
    output_max: int = 255

    def requant(self) -> tuple[int, int]:
        """(multiplier, shift) as computed by the native library."""
        m = ctypes.c_int32()
        s = ctypes.c_int32()
        L.check(L.lib().icv_requant_params(float(self.input_scale), float(self.kernel_scale),
                                           float(self.output_scale), ctypes.byref(m), ctypes.byref(s)),
                "icv_requant_params")
        return m.value, s.value


@dataclass
class PackedFilter:
    """Filter weights re-laid-out once for the device kernels (gemm.py:94-132)."""

    k_out: int
    kernel_elems: int
    in_channels: int
    nr: int
    dtype: torch.dtype            # compute dtype of the convolution this filter feeds
    params: ConvParams
    packed: torch.Tensor          # uint8 device buffer written by icv_pack_filter
    bias: torch.Tensor            # host copy of the caller's bias (float32 / int32)
    quant: QuantParams | None = None
    # pack_filter's own copy of the K x R x S x C weights (device, compute
    # dtype's source precision).  The reference PackedFilter likewise holds a
    # second copy of the weights (lane_weights, gemm.py:101-106); this one
    # backs the reference-layout views below and the GEMM baseline's 1x1
    # repack (im2col.py).  Never an alias of the caller's tensor, so editing
    # the caller's filter after packing changes nothing here.
    krsc: torch.Tensor | None = None

    @property
    def reduction_len(self) -> int:
        return self.kernel_elems * self.in_channels

    @property
    def n_tiles(self) -> int:
        return -(-self.k_out // self.nr)

    @property
    def device(self) -> torch.device:
        return self.packed.device

    def _krsc(self) -> torch.Tensor:
        if self.krsc is None:
            raise ValueError("this packed filter holds no weight copy (built by hand, not by pack_filter)")
        return self.krsc

    @property
    def weights(self) -> torch.Tensor:
        """(n_tiles, kernel_elems * in_channels, nr) column-tile panels, zero
        in the padded lanes: the reference's canonical packed layout
        (gemm.py:99-106, :153-157), on the device.  Built on first use."""
        cached = getattr(self, "_weights_view", None)
        if cached is None:
            k, rs, c, nr, nt = self.k_out, self.kernel_elems, self.in_channels, self.nr, self.n_tiles
            w = self._krsc().reshape(k, rs, c)
            lanes = torch.zeros((nt * nr, rs, c), dtype=w.dtype, device=w.device)
            lanes[:k] = w
            cached = lanes.reshape(nt, nr, rs, c).permute(0, 2, 3, 1).reshape(nt, rs * c, nr).contiguous()
            self._weights_view = cached
        return cached

    @property
    def lane_weights(self) -> torch.Tensor:
        """(kernel_elems * in_channels, n_tiles, nr): one reduction step across
        all column tiles (gemm.py:101-106, :158)."""
        cached = getattr(self, "_lane_view", None)
        if cached is None:
            cached = self.weights.permute(1, 0, 2).contiguous()
            self._lane_view = cached
        return cached

    def tile(self, jt: int) -> torch.Tensor:
        """(reduction_len, nr) panel of column tile jt; a view (gemm.py:116-118)."""
        return self.weights[jt]

    def lane_view(self) -> torch.Tensor:
        """(reduction_len, n_tiles, nr) reduction-step-major copy (gemm.py:120-124)."""
        return self.lane_weights

    def padded_bias(self) -> np.ndarray:
        """(n_tiles, nr) bias with zero in the padded lanes (gemm.py:128-132)."""
        pb = np.zeros((self.n_tiles, self.nr), dtype=np.float32 if self.dtype != torch.uint8 else np.int32)
        pb.reshape(-1)[: self.k_out] = self.bias.cpu().numpy()
        return pb


_W_DTYPES = (torch.float32, torch.bfloat16, torch.uint8)


def pack_filter(filt: FilterTensor, bias, params: ConvParams, tile: TileConfig, *,
                compute_dtype: torch.dtype | None = None, quant: QuantParams | None = None,
                device=None) -> PackedFilter:
    """Repack K x R x S x C weights for the device kernels (gemm.py:135-167).

    ``compute_dtype`` defaults to the filter's dtype: float32 selects the
    bit-exact float32 kernel, bfloat16 the tcgen05 kernel, uint8 the
    quantized tcgen05 kernel (``quant`` required).  ``bias`` is None (zeros),
    a float32 vector of length K (float paths) or an int32 vector (uint8).
    """
    if not filt.matches(params):
        raise ValueError("filter dimensions do not match params")                      # gemm.py:145-146
    compute_dtype = filt.dtype if compute_dtype is None else compute_dtype
    if compute_dtype not in _W_DTYPES:
        raise TypeError(f"unsupported compute dtype {compute_dtype}")
    if filt.dtype not in _W_DTYPES:
        raise TypeError(f"unsupported filter dtype {filt.dtype}")
    k = filt.k_out
    bias_dtype = torch.int32 if compute_dtype == torch.uint8 else torch.float32
    if bias is None:
        bias_t = torch.zeros(k, dtype=bias_dtype)
    else:
        bias_t = torch.as_tensor(bias) if not isinstance(bias, torch.Tensor) else bias
        if bias_t.dtype != bias_dtype or tuple(bias_t.shape) != (k,):
            kind = "int32" if bias_dtype == torch.int32 else "float32"
            raise ValueError(f"bias must be {kind} of length out_channels")               # gemm.py:164-165
        bias_t = bias_t.detach().clone().cpu()                                            # copied (:166)
    if compute_dtype == torch.uint8:
        if quant is None:
            raise ValueError("uint8 convolution needs QuantParams")
        if filt.dtype != torch.uint8:
            raise TypeError("uint8 convolution needs a uint8 filter")
    elif filt.dtype == torch.uint8:
        raise TypeError("float convolution needs a float filter")
    device = filt.data.device if device is None else torch.device(device)
    if device.type != "cuda":
        raise L.NativeLibraryError(f"filters are packed on a CUDA device (got {device}); there is no CPU fallback")
    # pack_filter's own copy (never an alias of the caller's tensor)
    w = filt.data.detach().to(device=device, copy=True)
    d = L.desc_of(params)
    nbytes = ctypes.c_int64()
    L.check(L.lib().icv_packed_filter_bytes(ctypes.byref(d), L.TORCH_TO_ICV[compute_dtype], ctypes.byref(nbytes)),
            "icv_packed_filter_bytes")
    packed = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
    bias_dev = bias_t.to(device) if bias is not None else None
    q = L.quant_of(quant)
    with torch.cuda.device(device):
        L.check(L.lib().icv_pack_filter(ctypes.byref(d), L.TORCH_TO_ICV[compute_dtype], L.TORCH_TO_ICV[w.dtype],
                                        L.ptr(w), L.ptr(bias_dev) if bias_dev is not None else None,
                                        ctypes.byref(q) if q is not None else None, L.ptr(packed),
                                        L.stream_of(device)),
                "icv_pack_filter")
    # keep the temporaries alive until the packing kernels have consumed them
    torch.cuda.current_stream(device).synchronize()
    return PackedFilter(k, params.kernel_elems, params.in_channels, tile.nr, compute_dtype, params, packed,
                        bias_t, quant, krsc=w)
