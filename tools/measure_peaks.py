"""Measure the peaks MEASURED_PEAKS.json lacks: dense int8
tensor throughput (torch._int_mm -> cuBLASLt, 8192^3, best of 10) and CUDA-core
fp32 (torch.matmul with TF32 off, 8192^3).  Library GEMMs are used for
calibration only.  Writes profiles/peaks_extra.json (read by bench.py)."""
import json
import os
import sys

import torch


def best_tflops(fn, flops, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = max(best, flops / (s.elapsed_time(e) * 1e-3) / 1e12)
    return best


def main():
    n = 8192
    dev = torch.device("cuda", 0)
    a8 = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev)
    b8 = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
    i8 = best_tflops(lambda: torch._int_mm(a8, b8), 2 * n ** 3)
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.randn(n, n, device=dev)
    b = torch.randn(n, n, device=dev)
    f32 = best_tflops(lambda: torch.matmul(a, b), 2 * n ** 3, reps=3)
    out = {"int8_tops": round(i8, 1), "fp32_tflops": round(f32, 2), "gemm": f"{n}^3",
           "how": "torch._int_mm int8 (cuBLASLt) best of 10; torch.matmul fp32 (TF32 off) best of 3; CUDA events",
           "gpu": torch.cuda.get_device_name(0)}
    print(json.dumps(out))
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "peaks_extra.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
