"""Pinned host <-> device copy rates on the box (H2D, D2H, both at once)."""
import torch

n = 12845056
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps):
        fn()
    en.record()
    torch.cuda.synchronize()
    return st.elapsed_time(en) / reps


def both():
    cur = torch.cuda.current_stream()
    e = torch.cuda.Event()
    e.record(cur)
    s1.wait_event(e)
    s2.wait_event(e)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
bi = timed(both)
print(f"H2D {n / h2d / 1e6:.1f} GB/s ({h2d * 1e3:.0f} us), D2H {n / d2h / 1e6:.1f} GB/s ({d2h * 1e3:.0f} us), "
      f"both concurrently {bi * 1e3:.0f} us")
