"""Batch-dimension data parallelism for the indirect convolution.

The operator shards naturally by image: the indirection-buffer entries,
accumulations and outputs of image n depend only on image n and on the
(replicated) filter (reference indirect.py:112-125), so there is no exchange
step in the data path.  Each rank owns a contiguous slice of the batch,
builds its own indirection buffer against its local shard (which equals the
full-batch buffer rows rebased by -n0*H*W*C, ZERO_REF kept), and writes its
own output shard.  The one collective is a broadcast of the packed filter
(and its folded epilogue constants) from the source rank, once per model
load, over NCCL on NVLink 5 / NVSwitch (gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .gemm import PackedFilter


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) image slice of rank `rank`; the first n % world
    ranks get one extra image.  Every image belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def broadcast_packed_filter(pf: PackedFilter, src: int = 0, group=None) -> PackedFilter:
    """Replicate the packed filter bytes from `src` to every rank in place
    (the only collective of the sharded convolution).  The host-side bias
    copy is broadcast too so every rank's PackedFilter is identical."""
    dist.broadcast(pf.packed, src=src, group=group)
    bias = pf.bias.to(pf.packed.device) if pf.packed.device.type == "cuda" else pf.bias
    dist.broadcast(bias, src=src, group=group)
    pf.bias = bias.cpu()
    return pf


def rebase_offsets(offsets: torch.Tensor, n0: int, image_elems: int) -> torch.Tensor:
    """Full-batch buffer rows -> the shard-local buffer of a rank whose first
    image is n0: subtract n0*H*W*C from every valid entry, keep ZERO_REF.
    (Used by tests to check that per-shard buffers equal the global one.)"""
    shift = n0 * image_elems
    return torch.where(offsets < 0, offsets, offsets - shift)
