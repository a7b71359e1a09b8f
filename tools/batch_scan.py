"""Time one cfg5 layer geometry at several batch sizes (synthetic data, L2
flushed): separates a per-launch fixed cost from the per-image cost.
    python tools/batch_scan.py s3b2_1x1a 64,128,256,512"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200.workloads import resnet50_layers  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    flush = bench.make_l2_flush(dev)
    for name in sys.argv[1].split(","):
        for batch in (int(b) for b in sys.argv[2].split(",")):
            _, shape, p = [t for t in resnet50_layers(batch) if t[0] == name][0]
            x = icv.NhwcTensor(shape, torch.randn(shape.numel, device=dev).to(torch.bfloat16))
            w = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels,
                                 torch.randn(p.out_channels * p.kernel_elems * p.in_channels, device=dev) * 0.05)
            tile = icv.TileConfig(mr=128)
            pf = icv.pack_filter(w, None, p, tile, compute_dtype=torch.bfloat16)
            zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16)
            o = icv.conv_output_shape(p, shape)
            ib = icv.init_indirection_buffer(x, zero, p, o, tile, per_image=True)
            y = icv.NhwcTensor.empty(o, dtype=torch.bfloat16, device=dev)
            t = bench.time_steps(lambda: icv.indirect_conv(x, pf, ib, p, tile, out=y), 9, 3, flush)
            print(f"{name:12s} N={batch:4d} {L.kernel_name(p, shape, torch.bfloat16):30s} "
                  f"{statistics.median(t) * 1e3:8.1f} us", flush=True)
            del x, w, pf, ib, y
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
