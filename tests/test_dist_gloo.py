"""Batch-sharded (data-parallel) path on the CPU with torch.distributed/gloo,
world_size 2: shard bookkeeping, the packed-filter broadcast (the only
collective of the sharded convolution) and the per-shard indirection buffer
(= the global buffer's rows rebased by -n0*H*W*C, ZERO_REF kept)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02129_b200.dist import broadcast_packed_filter, rebase_offsets, shard_range


def test_shard_range_partitions_every_image_once():
    for n in (1, 7, 64, 256):
        for world in (1, 2, 3, 4, 8):
            if world > n:
                continue
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, world, r)
                assert hi - lo in (n // world, n // world + 1)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1907_02129_b200 as icv
        from conftest import make_params
        from oracle import conv as oconv
        from oracle import ib as oib

        # 1. packed-filter broadcast: rank 0's bytes land on every rank
        p = make_params(r=3, s=3, pt=1, pl=1, c=8, k=6)
        if rank == 0:
            packed = torch.arange(512, dtype=torch.int64).to(torch.uint8)
            bias = torch.linspace(-1, 1, 6)
        else:
            packed = torch.zeros(512, dtype=torch.uint8)
            bias = torch.zeros(6)
        pf = icv.PackedFilter(6, 9, 8, 8, torch.bfloat16, p, packed, bias)
        broadcast_packed_filter(pf, src=0)
        ok_bcast = torch.equal(pf.packed, torch.arange(512, dtype=torch.int64).to(torch.uint8)) and \
            torch.allclose(pf.bias, torch.linspace(-1, 1, 6))

        # 2. per-shard buffer == rebased global rows; sharded conv == global conv
        n, h, w, c = 5, 7, 6, 8
        x = np.random.default_rng(3).uniform(-1, 1, n * h * w * c).astype(np.float32)
        wt = np.random.default_rng(4).uniform(-1, 1, 6 * 9 * c).astype(np.float32)
        oh, ow = oib.out_hw(p, h, w)
        lo, hi = shard_range(n, world, rank)
        full = oib.compute_offsets((n, h, w, c), p, oh, ow, n, 4)
        refs_full = oconv.pixel_refs(full, n * oh * ow)
        local = oib.compute_offsets((hi - lo, h, w, c), p, oh, ow, hi - lo, 4)
        refs_local = oconv.pixel_refs(local, (hi - lo) * oh * ow)
        rebased = rebase_offsets(torch.from_numpy(refs_full[lo * oh * ow:hi * oh * ow]), lo, h * w * c).numpy()
        ok_ib = np.array_equal(refs_local, rebased)
        y_local = oconv.indirect_conv_f32(x[lo * h * w * c:hi * h * w * c], np.zeros(c, np.float32), local, p, wt,
                                          None, hi - lo, oh, ow)
        # gather only to check the result; the data path itself has no collective
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([y_local.size], dtype=torch.int64))
        maxn = int(max(s.item() for s in sizes))
        buf = torch.zeros(maxn)
        buf[:y_local.size] = torch.from_numpy(y_local.reshape(-1))
        parts = [torch.zeros(maxn) for _ in range(world)]
        dist.all_gather(parts, buf)
        y = np.concatenate([parts[r][:int(sizes[r].item())].numpy() for r in range(world)])
        y_ref = oconv.indirect_conv_f32(x, np.zeros(c, np.float32), full, p, wt, None, n, oh, ow)
        ok_conv = y.tobytes() == y_ref.reshape(-1).tobytes()
        q.put((rank, ok_bcast, ok_ib, ok_conv))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_path():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok_bcast, ok_ib, ok_conv in results:
        assert ok_bcast, f"rank {rank}: packed filter not replicated"
        assert ok_ib, f"rank {rank}: shard buffer != rebased global rows"
        assert ok_conv, f"rank {rank}: sharded convolution != global convolution"
