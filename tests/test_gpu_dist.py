"""The batch-sharded CUDA path on the one GPU of the test box.

* The native NCCL communicator (icv_nccl_*): init_all / init_rank over one
  device, in-place broadcast, communicator size.
* Two ranks, both on cuda:0 (torch.distributed over gloo for the host-side
  coordination; the ranks' kernels never wait on each other): rank 0 packs
  the filter and broadcasts it, every rank convolves its own image shard
  through ShardedIndirectConv, and the gathered shards equal rank 0's
  single-rank full-batch output BYTE FOR BYTE, for cfg2 (bf16) and cfg4
  (uint8).  Per-image independence: reference indirect.py:112-125.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def test_native_nccl_single_device_broadcast():
    import paper_1907_02129_b200 as icv

    assert icv.NcclComm.version() >= 22000
    (c,) = icv.NcclComm.init_all([0])
    t = torch.arange(1000, dtype=torch.int32, device="cuda:0")
    c.broadcast_(t, 0)
    torch.cuda.synchronize()
    assert c.size() == 1 and torch.equal(t.cpu(), torch.arange(1000, dtype=torch.int32))
    c.close()
    r = icv.NcclComm.init_rank(0, 1, icv.NcclComm.unique_id(), "cuda:0")
    u = torch.full((77,), 5, dtype=torch.uint8, device="cuda:0")
    r.broadcast_(u, 0)
    torch.cuda.synchronize()
    assert r.size() == 1 and int(u.sum()) == 5 * 77
    r.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(name, lo, hi, device):
    import paper_1907_02129_b200 as icv
    from paper_1907_02129_b200.workloads import CONFIGS

    w = CONFIGS[name]
    s = w.in_shape
    dt = {"bf16": torch.bfloat16, "u8": torch.uint8}[w.dtype]
    x = icv.NhwcTensor(icv.Shape4(hi - lo, s.h, s.w, s.c), torch.from_numpy(w.input_host(lo, hi)).to(device).to(dt))
    qp = None
    if w.quant is not None:
        q = w.quant
        qp = icv.QuantParams(q.input_zero_point, q.input_scale, q.kernel_zero_point, q.kernel_scale,
                             q.output_zero_point, q.output_scale, q.output_min, q.output_max)
    return w, x, dt, qp


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1907_02129_b200 as icv
        from paper_1907_02129_b200.workloads import CONFIGS

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        w0 = CONFIGS[name]
        n = w0.in_shape.n
        lo, hi = icv.shard_range(n, world, rank)
        w, x, dt, qp = _problem(name, lo, hi, dev)
        p = w.params
        tile = icv.TileConfig(mr=128)
        filt, bias = None, w.bias_host()
        if rank == 0:
            filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                                    torch.from_numpy(w.filter_host()).to(dev).to(dt))
        pf = icv.replicate_filter(filt, None if bias is None else torch.from_numpy(bias), p, tile, rank=rank,
                                  device=dev, compute_dtype=dt, quant=qp)
        op = icv.ShardedIndirectConv(p, tile, pf)
        y_local = op(x).data.cpu().view(torch.uint8).numpy()
        op(x)   # a second call reuses the cached buffer
        hits = op.cache.stats.hits
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, y_local.tobytes()))
        ok = None
        if rank == 0:
            wf, xf, _, _ = _problem(name, 0, n, dev)
            pff = icv.pack_filter(icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                                                   torch.from_numpy(w.filter_host()).to(dev).to(dt)),
                                  None if bias is None else torch.from_numpy(bias), p, tile, quant=qp)
            full = icv.ShardedIndirectConv(p, tile, pff)(xf).data.cpu().view(torch.uint8).numpy().tobytes()
            joined = b"".join(b for _, _, b in sorted(parts))
            ok = (joined == full, [(a, b) for a, b, _ in sorted(parts)], len(full))
        q.put((rank, ok, hits, bytes(pf.packed.cpu().numpy()[:64])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_two_ranks_on_one_gpu_shard_byte_identical(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = sorted(q.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    (_, ok, hits0, head0), (_, _, hits1, head1) = results
    same, ranges, nbytes = ok
    assert ranges == [(0, 32 if name == "cfg2" else 64), (32 if name == "cfg2" else 64, 64 if name == "cfg2" else 128)]
    assert same, f"{name}: gathered shards differ from the single-rank output ({nbytes} bytes)"
    assert head0 == head1, "packed filter not replicated"
    assert hits0 == hits1 == 1
