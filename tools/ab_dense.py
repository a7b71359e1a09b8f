import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1907_02129_b200 import _lib as L
from paper_1907_02129_b200.stack import ResNet50Stack
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
stack = ResNet50Stack(device=dev)
flush = bench.make_l2_flush(dev)
names = sys.argv[1].split(",")
by = {l.name: l for l in stack.layers}
for cs in [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1,2").split(",")]:
    L.set_tuning("dense_cs", cs)
    for n in names:
        l = by[n]
        t = bench.time_steps(lambda: stack.run_layer(l), 7, 2, flush)
        print(f"cs={cs} {n:12s} {L.kernel_name(l.params, l.input.shape, torch.bfloat16):32s} {statistics.median(t)*1e3:8.1f} us", flush=True)
