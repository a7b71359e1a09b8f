"""cfg5: time the ResNet-50 conv stack (N=256 by default) layer by layer.

    python tools/time_stack.py [batch] [--json out.json]

Per layer: median CUDA-event time over the timed passes, TFLOP/s, the
roofline time min-bound = max(FLOPs / bf16 peak, compulsory bytes / HBM BW)
and the achieved fraction of it; end to end = total FLOPs / median pass time
(max pool included, and reported separately).
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_02129_b200 import _lib as L  # noqa: E402
from paper_1907_02129_b200.stack import ResNet50Stack  # noqa: E402


def peaks():
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    bf16, hbm = 1638.3, 6545.3
    try:
        m = json.load(open(path))
        bf16 = float(m.get("bf16_tflops", bf16))
        hbm = float(m.get("hbm_gbs", hbm))
    except (OSError, ValueError):
        pass
    return bf16, hbm


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    batch = int(args[0]) if args else 256
    out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    passes = 5
    stack = ResNet50Stack(batch=batch, device="cuda")
    for _ in range(2):
        stack.run()
    torch.cuda.synchronize()
    totals, pools, per = [], [], []
    for _ in range(passes):
        t, pool, layers = stack.timed_run()
        totals.append(t)
        pools.append(pool)
        per.append(layers)
    bf16, hbm = peaks()
    rows = []
    for i, layer in enumerate(stack.layers):
        ms = statistics.median(p[i] for p in per)
        bound_ms = max(layer.flops / (bf16 * 1e9), layer.compulsory_bytes / (hbm * 1e6))
        rows.append({
            "layer": layer.name, "kernel": L.kernel_name(layer.params, layer.input.shape, torch.bfloat16),
            "us": round(ms * 1e3, 2), "tflops": round(layer.flops / ms / 1e9, 1),
            "roofline_us": round(bound_ms * 1e3, 2), "frac": round(bound_ms / ms, 3),
            "bound": "tensor" if layer.flops / (bf16 * 1e9) >= layer.compulsory_bytes / (hbm * 1e6) else "hbm",
        })
    total = statistics.median(totals)
    pool = statistics.median(pools)
    conv_ms = sum(r["us"] for r in rows) / 1e3
    roof_ms = sum(r["roofline_us"] for r in rows) / 1e3
    for r in rows:
        print(f"{r['layer']:12s} {r['kernel']:24s} {r['us']:9.1f} us {r['tflops']:8.1f} TFLOP/s "
              f"roofline {r['roofline_us']:8.1f} us ({r['bound']}) frac {r['frac']:.2f}")
    summary = {
        "workload": f"cfg5_resnet50_conv_stack_bf16_n{batch}", "layers": len(rows),
        "gflop": round(stack.flops / 1e9, 1), "total_ms": round(total, 3), "maxpool_ms": round(pool, 3),
        "conv_ms": round(conv_ms, 3), "tflops_end_to_end": round(stack.flops / total / 1e9, 1),
        "tflops_convs_only": round(stack.flops / conv_ms / 1e9, 1),
        "sum_roofline_ms": round(roof_ms, 3), "frac_of_sum_roofline": round(roof_ms / conv_ms, 3),
        "peaks": {"bf16_tflops": bf16, "hbm_gbs": hbm},
    }
    print(json.dumps(summary))
    if out_json:
        json.dump({"summary": summary, "layers": rows}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
