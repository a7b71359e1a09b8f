"""Batch-dimension data parallelism for the indirect convolution
(SURVEY.md §8(e)).

The operator shards naturally by image: the indirection-buffer entries,
accumulations and outputs of image n depend only on image n and on the
(replicated) filter (reference indirect.py:112-125), so there is no
exchange step in the data path.  Each rank owns a contiguous slice of the
batch (``shard_range``), builds its own indirection buffer against its
local shard (which equals the full-batch buffer's rows rebased by
-n0*H*W*C, ZERO_REF kept: ``rebase_offsets``), and writes its own output
shard.  The one collective is a broadcast of the packed filter (and its
folded epilogue constants) from the source rank, once per model load: over
NCCL on NVLink 5 / NVSwitch through the native library's ``icv_nccl_*``
entry points (``NcclComm``), or through any torch.distributed group (gloo
in the CPU tests).

Pieces:
  * ``NcclComm``           -- the native NCCL communicator (init per rank or
                              all local GPUs in one process), broadcast.
  * ``replicate_filter``   -- pack on the source rank, broadcast to all.
  * ``ShardedIndirectConv``-- one rank's operator: replicated packed filter,
                              an IndirectionCache over the local shard,
                              ``indirect_conv`` into the local output shard.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib as L
from .gemm import PackedFilter, QuantParams, TileConfig, pack_filter
from .ib_cache import IndirectionCache
from .indirect import indirect_conv, make_zero_row
from .tensors import ConvParams, FilterTensor, NhwcTensor


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) image slice of rank `rank`; the first n % world
    ranks get one extra image.  Every image belongs to exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


class NcclComm:
    """A NCCL communicator owned by the native library (include/icv.h
    ``icv_nccl_*``; libnccl.so.2 is loaded at run time)."""

    UNIQUE_ID_BYTES = 128

    def __init__(self, handle: int, rank: int, world: int, device: torch.device):
        self.handle = ctypes.c_void_p(handle)
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def version() -> int:
        v = ctypes.c_int32()
        L.check(L.lib().icv_nccl_version(ctypes.byref(v)), "icv_nccl_version")
        return int(v.value)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(NcclComm.UNIQUE_ID_BYTES)
        L.check(L.lib().icv_nccl_unique_id(buf), "icv_nccl_unique_id")
        return buf.raw

    @classmethod
    def init_rank(cls, rank: int, world: int, unique_id: bytes, device) -> "NcclComm":
        """Join a ``world``-rank communicator (one process per GPU) on
        ``device``; ``unique_id`` comes from rank 0's ``unique_id()``."""
        device = torch.device(device)
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), NcclComm.UNIQUE_ID_BYTES)
        with torch.cuda.device(device):
            L.check(L.lib().icv_nccl_init_rank(ctypes.byref(h), world, buf, rank), "icv_nccl_init_rank")
        return cls(h.value, rank, world, device)

    @classmethod
    def init_all(cls, devices: list[int]) -> list["NcclComm"]:
        """One communicator per local GPU, all from this process."""
        n = len(devices)
        hs = (ctypes.c_void_p * n)()
        devs = (ctypes.c_int32 * n)(*devices)
        L.check(L.lib().icv_nccl_init_all(hs, n, devs), "icv_nccl_init_all")
        return [cls(hs[i], i, n, torch.device("cuda", devices[i])) for i in range(n)]

    @classmethod
    def from_process_group(cls, device, group=None) -> "NcclComm":
        """Communicator over the ranks of an initialized torch.distributed
        group; the unique id travels through that group (a host-side object
        broadcast), the data never does."""
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group, device=torch.device(device) if dist.get_backend(group) == "nccl"
                                   else None)
        return cls.init_rank(rank, world, obj[0], device)

    def size(self) -> int:
        n = ctypes.c_int32()
        L.check(L.lib().icv_nccl_comm_size(self.handle, ctypes.byref(n)), "icv_nccl_comm_size")
        return int(n.value)

    def broadcast_(self, t: torch.Tensor, root: int = 0) -> torch.Tensor:
        """In-place broadcast of a contiguous device tensor from ``root``,
        stream-ordered on the current stream of its device."""
        if not t.is_contiguous() or t.device.type != "cuda":
            raise ValueError("broadcast_ needs a contiguous CUDA tensor")
        with torch.cuda.device(t.device):
            L.check(L.lib().icv_nccl_broadcast(None, L.ptr(t), t.numel() * t.element_size(), root, self.handle,
                                               L.stream_of(t.device)), "icv_nccl_broadcast")
        return t

    def close(self) -> None:
        if self.handle:
            L.check(L.lib().icv_nccl_destroy(self.handle), "icv_nccl_destroy")
            self.handle = ctypes.c_void_p()


def broadcast_packed_filter(pf: PackedFilter, src: int = 0, group=None, comm: NcclComm | None = None
                            ) -> PackedFilter:
    """Replicate the packed filter bytes (weights + folded epilogue
    constants) from `src` to every rank in place -- the only collective of
    the sharded convolution.  With ``comm`` it runs on the native NCCL
    communicator; otherwise on a torch.distributed group.  The host-side
    bias copy is broadcast too, so every rank's PackedFilter is identical."""
    if comm is not None:
        comm.broadcast_(pf.packed, src)
        bias = pf.bias.to(pf.packed.device)
        comm.broadcast_(bias, src)
        pf.bias = bias.cpu()
        return pf
    if dist.get_backend(group) == "nccl":       # device transport
        dist.broadcast(pf.packed, src=src, group=group)
        bias = pf.bias.to(pf.packed.device)
        dist.broadcast(bias, src=src, group=group)
        pf.bias = bias.cpu()
        return pf
    # a host-transport group (gloo): stage device bytes through host memory
    host = pf.packed.cpu()
    dist.broadcast(host, src=src, group=group)
    if pf.packed.device.type == "cuda":
        pf.packed.copy_(host)
    else:
        pf.packed = host
    bias = pf.bias.cpu().clone()
    dist.broadcast(bias, src=src, group=group)
    pf.bias = bias
    return pf


def empty_packed_filter(params: ConvParams, tile: TileConfig, compute_dtype: torch.dtype, device,
                        quant: QuantParams | None = None) -> PackedFilter:
    """A receive buffer with the exact layout pack_filter would produce on
    this rank (icv_packed_filter_bytes), to be filled by a broadcast."""
    d = L.desc_of(params)
    nbytes = ctypes.c_int64()
    L.check(L.lib().icv_packed_filter_bytes(ctypes.byref(d), L.TORCH_TO_ICV[compute_dtype], ctypes.byref(nbytes)),
            "icv_packed_filter_bytes")
    bias_dtype = torch.int32 if compute_dtype == torch.uint8 else torch.float32
    return PackedFilter(params.out_channels, params.kernel_elems, params.in_channels, tile.nr, compute_dtype, params,
                        torch.empty(nbytes.value, dtype=torch.uint8, device=device),
                        torch.zeros(params.out_channels, dtype=bias_dtype), quant, krsc=None)


def replicate_filter(filt: FilterTensor | None, bias, params: ConvParams, tile: TileConfig, *, rank: int,
                     device, compute_dtype: torch.dtype | None = None, quant: QuantParams | None = None,
                     src: int = 0, comm: NcclComm | None = None, group=None) -> PackedFilter:
    """Pack the filter on the source rank (the only rank that needs the
    weights) and broadcast the packed bytes to every rank."""
    if rank == src:
        if filt is None:
            raise ValueError("the source rank must supply the filter")
        pf = pack_filter(filt, bias, params, tile, compute_dtype=compute_dtype, quant=quant, device=device)
    else:
        if compute_dtype is None:
            raise ValueError("non-source ranks must name the compute dtype")
        pf = empty_packed_filter(params, tile, compute_dtype, device, quant)
    return broadcast_packed_filter(pf, src, group=group, comm=comm)


class ShardedIndirectConv:
    """One rank of a batch-sharded indirect convolution.

    Holds the replicated packed filter and an ``IndirectionCache`` over the
    rank's local input shard (built on first use, reused while the shard
    stays at the same location -- PAPER.md §2.3); ``__call__`` convolves the
    local shard into the local output shard with no communication."""

    def __init__(self, params: ConvParams, tile: TileConfig, pf: PackedFilter, *, per_image: bool = True,
                 index_dtype: torch.dtype = torch.int64):
        self.params, self.tile, self.pf = params, tile, pf
        fill = pf.quant.input_zero_point if (pf.quant is not None and pf.dtype == torch.uint8) else 0
        self.zero_row = make_zero_row(params.in_channels, dtype=pf.dtype, device=pf.device, fill=fill)
        self.cache = IndirectionCache(params, tile, self.zero_row, index_dtype=index_dtype, per_image=per_image)

    def __call__(self, x_local: NhwcTensor, out: NhwcTensor | None = None, algorithm: str = "auto") -> NhwcTensor:
        ib = self.cache.get(x_local)
        return indirect_conv(x_local, self.pf, ib, self.params, self.tile, out=out, algorithm=algorithm)


def rebase_offsets(offsets: torch.Tensor, n0: int, image_elems: int) -> torch.Tensor:
    """Full-batch buffer rows -> the shard-local buffer of a rank whose first
    image is n0: subtract n0*H*W*C from every valid entry, keep ZERO_REF.
    (Used by tests to check that per-shard buffers equal the global one.)"""
    shift = n0 * image_elems
    return torch.where(offsets < 0, offsets, offsets - shift)
