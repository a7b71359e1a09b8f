"""The paper's evaluation on B200 (§4, Figures 5-6, Tables 2-3):
every shape of the ResNet-18 / SqueezeNet 1.0 (and ResNet-50) suites through
the GPU harness -- indirect (default kernel), indirect_gather (the IB-gather
mainloop), gemm_based (im2row + dense GEMM) and gemm_only -- in bf16 at a
batch that fills the GPU, with per-layer TFLOP/s, roofline fraction, gates,
and the per-class geomean speedups.

    python tools/suite_table.py [--batch 64] [--reps 10] [--out profiles/r02_suites]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1907_02129_b200 import harness  # noqa: E402
from paper_1907_02129_b200.analysis import b200_lambda  # noqa: E402
from paper_1907_02129_b200.suites import load_shape_suite  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--suites", default="resnet18,squeezenet10,resnet50")
    ap.add_argument("--out", default="profiles/r02_suites")
    args = ap.parse_args()
    lam = b200_lambda("bf16")
    summary = {"batch": args.batch, "dtype": "bf16", "lambda_b200": round(lam, 1), "suites": {}}
    md = [f"# Suites on B200 (bf16, batch {args.batch}, median of {args.reps} interleaved reps, CUDA events)", ""]
    for name in args.suites.split(","):
        suite = load_shape_suite(name)
        res = harness.run_benchmark(suite, variants=harness.VARIANTS, reps=args.reps, warmup=3, lam=lam,
                                    dtype=torch.bfloat16, batch=args.batch, min_sample_s=2e-4)
        harness.emit_report(res, "json", f"{args.out}_{name}.json")
        table = harness.speedup_table(res)
        summary["suites"][name] = table
        md += [f"## {name}", "", "| shape | indirect kernel | indirect TFLOP/s | frac | gather TFLOP/s | gemm_based | "
               "gemm_only | indirect / gemm_based | indirect / gemm_only |", "|---|---|---|---|---|---|---|---|---|"]
        by = {(r.shape, r.variant): r for r in res.reports}
        for spec in suite:
            r = by.get((spec.name, "indirect"))
            if r is None:
                continue
            g = by.get((spec.name, "indirect_gather"))
            gb = by.get((spec.name, "gemm_based"))
            go = by.get((spec.name, "gemm_only"))
            tf = lambda x: f"{x.median_gflops / 1e3:.1f}" if x else "-"   # noqa: E731
            sp = lambda x: f"{x.median_time_s / r.median_time_s:.2f}x" if x else "-"   # noqa: E731
            md.append(f"| {spec.name} | {r.kernel} | {tf(r)} | {r.roofline_frac:.2f} ({r.bound}) | {tf(g)} | {tf(gb)} "
                      f"| {tf(go)} | {sp(gb)} | {sp(go)} |")
        md += ["", "Geomean speedup of indirect by class (percent): " + json.dumps(table), ""]
        print(name, json.dumps(table), flush=True)
    with open(f"{args.out}.json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(f"{args.out}.md", "w") as f:
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
