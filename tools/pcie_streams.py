"""H2D / D2H rate of one 12.8 MB pinned copy split over k streams (copy engines)."""
import torch

n = 12845056
dev = torch.device("cuda", 0)
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
streams = [torch.cuda.Stream() for _ in range(8)]


def run(k, h2d=True, reps=20):
    parts = [(n * i // k, n * (i + 1) // k) for i in range(k)]

    def step():
        cur = torch.cuda.current_stream()
        e = torch.cuda.Event()
        e.record(cur)
        for i, (a, b) in enumerate(parts):
            s = streams[i]
            s.wait_event(e)
            with torch.cuda.stream(s):
                if h2d:
                    d[a:b].copy_(h[a:b], non_blocking=True)
                else:
                    h[a:b].copy_(d[a:b], non_blocking=True)
        for i in range(k):
            cur.wait_stream(streams[i])

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(reps):
        step()
    en.record()
    torch.cuda.synchronize()
    ms = st.elapsed_time(en) / reps
    print(f"{'H2D' if h2d else 'D2H'} split over {k} streams: {ms * 1e3:6.0f} us = {n / ms / 1e6:5.1f} GB/s")


for k in (1, 2, 4, 8):
    run(k, True)
for k in (1, 2, 4):
    run(k, False)
