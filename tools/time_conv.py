"""Median CUDA-event time of each config's convolution (L2 flushed between
iterations) plus a sampled-pixel correctness check; for A/B-ing variants."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402

# plan knobs for the run: ICV_KNOBS="cluster=2,u8_bn=256"
for _kv in filter(None, os.environ.get("ICV_KNOBS", "").split(",")):
    icv._lib.set_tuning(_kv.split("=")[0], int(_kv.split("=")[1]))


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    names = sys.argv[1:] or ["cfg2", "cfg3b", "cfg4"]
    dev = torch.device("cuda", 0)
    flush_l2 = bench.make_l2_flush(dev)
    for name in names:
        w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, CONFIGS[name].in_shape.n, dev,
                                                        per_image=os.environ.get("ICV_IB", "per-image") == "per-image")
        if os.environ.get("ICV_NONCANONICAL"):
            ib.canonical = False
        t = bench.time_steps(lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y), 50, 5,
                             flush_l2)
        ms = statistics.median(t)
        ok = ""
        if w.dtype == "bf16" and not os.environ.get("ICV_NO_GATE"):
            ok = bench.conv_gate(w, xh, ib, y)["normwise_rel_err"]
        kname = icv._lib.kernel_name(w.params, w.in_shape, x.dtype)
        print(f"{name:6s} {ms * 1e3:8.2f} us  {w.flops / ms / 1e9:8.1f} TFLOP/s  gate={ok}  [{kname}]")
        del x, pf, ib, y


if __name__ == "__main__":
    main()
