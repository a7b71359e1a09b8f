"""paper_1907_02129_b200 — B200-native indirect convolution (arXiv 1907.02129).

A drop-in for the hot path of the reference package ``convbench``
(/root/reference/pkg/src/convbench/__init__.py:31-49): the same names for
indirection-buffer setup, filter packing and indirect convolution, with all
compute in hand-written sm_100a kernels behind the C ABI of ``libicv.so``
(include/icv.h).  Tensors are torch tensors in device memory; torch is used
for allocation, streams and torch.distributed only.
"""

from .dist import NcclComm, ShardedIndirectConv, broadcast_packed_filter, replicate_filter, shard_range
from .errors import InvalidGeometryError, NativeLibraryError, StaleBufferError, UnsupportedError
from .gemm import PackedFilter, QuantParams, TileConfig, pack_filter
from .ib_cache import CacheStats, IndirectionCache
from .im2col import PatchMatrix, build_patch_matrix, gemm_conv, gemm_only
from .indirect import (
    ZERO_REF,
    IndirectionBuffer,
    indirect_conv,
    indirect_gemm_microkernel,
    init_indirection_buffer,
    make_zero_row,
    rebind_input,
    update_for_batch_growth,
)
from .tensors import (
    ConvParams,
    FilterTensor,
    NhwcTensor,
    Shape4,
    conv_output_shape,
    filter_fill_random,
    tensor_fill_random,
    tensor_fill_sequential,
)

__version__ = "0.1.0"

__all__ = [
    "NcclComm", "ShardedIndirectConv", "broadcast_packed_filter", "replicate_filter", "shard_range",
    "ZERO_REF", "CacheStats", "ConvParams", "FilterTensor", "IndirectionCache", "PatchMatrix", "build_patch_matrix", "gemm_conv", "gemm_only", "IndirectionBuffer", "InvalidGeometryError",
    "NativeLibraryError", "NhwcTensor", "PackedFilter", "QuantParams", "Shape4", "StaleBufferError",
    "TileConfig", "UnsupportedError", "conv_output_shape", "filter_fill_random", "indirect_conv",
    "indirect_gemm_microkernel", "init_indirection_buffer", "make_zero_row", "pack_filter", "rebind_input", "tensor_fill_random",
    "tensor_fill_sequential", "update_for_batch_growth",
]
