"""Where the per-step event time goes: one conv between events after an L2
flush (the bench's protocol) vs 100 back-to-back convs (queue kept full, no
flush) vs the same problem at batch 1 (fixed cost), for a config."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1907_02129_b200 as icv  # noqa: E402


def main():
    from paper_1907_02129_b200.workloads import CONFIGS

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    dev = torch.device("cuda", 0)
    flush = bench.make_l2_flush(dev)
    for nimg in (CONFIGS[name].in_shape.n, 1):
        w, x, xh, pf, ib, y, tile = bench.setup_problem(name, 0, nimg, dev)
        fn = lambda: icv.indirect_conv(x, pf, ib, w.params, tile, out=y)  # noqa: E731
        t = bench.time_steps(fn, 50, 5, flush)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(100):
            fn()
        e.record()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        for _ in range(5):
            g.replay()
        e2.record()
        torch.cuda.synchronize()
        print(f"{name} n={nimg}: flushed step median {statistics.median(t) * 1e3:.2f} us; "
              f"back-to-back {s.elapsed_time(e) * 10:.2f} us/launch; graph {s2.elapsed_time(e2) * 10:.2f} us/launch")


if __name__ == "__main__":
    main()
