"""Indirection-buffer lifecycle for a framework operator.

The paper keeps one indirection buffer per convolution operator and
reinitializes it only when needed (§2.3; reference
indirect.py:167-212): a new input *location* means a complete
re-initialization (``rebind_input``), a larger batch at the same location
means building only the new part (``update_for_batch_growth``), a smaller
batch is served by logical truncation, and a new input geometry means a new
buffer.  ``IndirectionCache`` applies exactly those rules to the tensors an
operator sees call after call, and counts what it did.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .gemm import TileConfig
from .indirect import (IndirectionBuffer, _same_binding, init_indirection_buffer, rebind_input,
                       update_for_batch_growth)
from .tensors import ConvParams, NhwcTensor, conv_output_shape


@dataclass
class CacheStats:
    hits: int = 0          # same binding, batch already covered (incl. logical truncation)
    builds: int = 0        # first buffer, or a new geometry / dtype / device
    rebinds: int = 0       # same geometry, new input location: complete re-initialization
    growths: int = 0       # same location, more images: only the new part built


class IndirectionCache:
    """One operator's indirection buffer, kept valid across calls.

    ``get(input, batch)`` returns a buffer bound to ``input`` that covers at
    least ``batch`` images (default: all of ``input``); pass the same
    ``batch`` to ``indirect_conv``.  ``zero_row`` is shared read-only
    (indirect.py:42) and fixes the dtype and device: an input of another
    dtype or device raises ValueError (as init_indirection_buffer does).
    Every call is counted exactly once in ``stats``."""

    def __init__(self, params: ConvParams, tile: TileConfig, zero_row: torch.Tensor, *,
                 index_dtype: torch.dtype = torch.int64, per_image: bool = False):
        self.params = params
        self.tile = tile
        self.zero_row = zero_row
        self.index_dtype = index_dtype
        self.per_image = per_image
        self.ib: IndirectionBuffer | None = None
        self.stats = CacheStats()

    def get(self, input: NhwcTensor, batch: int | None = None) -> IndirectionBuffer:
        batch = input.shape.n if batch is None else batch
        if not 1 <= batch <= input.shape.n:
            raise ValueError("batch must be within the input tensor's batch")
        ib = self.ib
        if ib is None or ib.in_shape != input.shape or ib.zero_row is not self.zero_row:
            # first call, or a new geometry (a differently sized tensor is a new location too)
            out_shape = conv_output_shape(self.params, input.shape)
            self.ib = init_indirection_buffer(input, self.zero_row, self.params, out_shape, self.tile, batch=batch,
                                              index_dtype=self.index_dtype, per_image=self.per_image)
            self.stats.builds += 1
            return self.ib
        if not _same_binding(ib.input_data, input.data):                                  # PAPER.md §2.3
            # complete re-initialization at the new location, for the larger of
            # the two batches (the zero row is unchanged: no re-scan of it)
            out_shape = conv_output_shape(self.params, input.shape)
            self.ib = init_indirection_buffer(input, self.zero_row, self.params, out_shape, self.tile,
                                              batch=max(batch, ib.batch), index_dtype=self.index_dtype,
                                              per_image=self.per_image, _zero_facts=(ib.zero_is_zero, ib.zero_fill_byte))
            self.stats.rebinds += 1
            return self.ib
        if batch > ib.batch:                                                              # indirect.py:167-193
            self.ib = update_for_batch_growth(ib, batch)
            self.stats.growths += 1
            return self.ib
        self.stats.hits += 1
        return ib
