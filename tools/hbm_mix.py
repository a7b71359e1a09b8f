"""HBM bandwidth by read:write mix on one B200 (what an output-heavy layer can
expect): write-only fill, 1:1 copy, 1:4 (read 1 byte, write 4: the ResNet-50
1x1 expansions' ratio) and 4:1 (a sum over 4 rows).  CUDA events, best of 10, L2 flushed by the
sheer size (1 GiB buffers)."""
import torch


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return min(ts)


def main():
    n = 1 << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    a.fill_(1)
    t = best(lambda: a.fill_(3))
    print(f"write-only fill      {n / t / 1e9:8.1f} GB/s")
    t = best(lambda: b.copy_(a))
    print(f"copy 1:1 (r+w)       {2 * n / t / 1e9:8.1f} GB/s")
    q = n // 4
    src = a[:q].view(q // 128, 1, 128)
    dst = b.view(q // 128, 4, 128)
    t = best(lambda: dst.copy_(src.expand(q // 128, 4, 128)))
    print(f"1:4 read:write       {(q + n) / t / 1e9:8.1f} GB/s")
    f = a.view(torch.float32)
    t = best(lambda: torch.sum(f.view(4, -1), 0))
    print(f"4:1 read:write       {(n + n // 4) / t / 1e9:8.1f} GB/s")

if __name__ == "__main__":
    main()
