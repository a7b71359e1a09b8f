"""The GPU benchmark harness (harness.py) end to end on small shapes:
gates against the device direct convolution (bit-exact float32, rel 1e-2
bf16), interleaved reps, nearest-rank quantiles, skip rule, CSV / JSON
reports that round-trip, and the CLI's exit codes; plus the device
direct_conv itself against the oracle."""

import json

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from oracle import conv as oconv
from paper_1907_02129_b200 import cli, harness
from paper_1907_02129_b200.reference import direct_conv
from paper_1907_02129_b200.suites import ConvShapeSpec, load_shape_suite

pytestmark = pytest.mark.gpu


def _spec(name, r, stride, pad, c, k, hw, dil=1):
    p = icv.ConvParams(r, r, stride_h=stride, stride_w=stride, dilation_h=dil, dilation_w=dil, pad_top=pad,
                       pad_left=pad, pad_bottom=pad, pad_right=pad, in_channels=c, out_channels=k)
    return ConvShapeSpec(name, icv.Shape4(1, hw, hw, c), p)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_device_direct_conv_matches_oracle(dt):
    s = _spec("t", 3, 2, 1, 16, 24, 11, dil=1)
    x = icv.tensor_fill_random(icv.Shape4(2, 11, 11, 16), 3, dtype=dt)
    f = icv.filter_fill_random(s.params, 4, dtype=dt)
    b = np.random.default_rng(5).uniform(-1, 1, 24).astype(np.float32)
    y = direct_conv(x, f, torch.from_numpy(b), s.params).numpy()
    ref = oconv.direct_conv_f32(x.data.float().cpu().numpy().reshape(2, 11, 11, 16), f.data.float().cpu().numpy(),
                                b, s.params)
    assert y.tobytes() == ref.reshape(-1).tobytes()


def test_run_benchmark_f32_bit_exact_and_reports(tmp_path):
    suite = [_spec("a3x3", 3, 1, 1, 16, 24, 12), _spec("b1x1", 1, 1, 0, 32, 16, 9), _spec("c3x3s2", 3, 2, 1, 8, 8, 13)]
    res = harness.run_benchmark(suite, variants=harness.VARIANTS, reps=3, warmup=1, min_sample_s=1e-4)
    got = {(r.shape, r.variant) for r in res.reports}
    assert ("b1x1", "gemm_only") not in got and [s.variant for s in res.skipped] == ["gemm_only"]
    assert len(got) == 3 * 4 - 1
    for r in res.reports:
        assert len(r.runs_s) == 3 and r.q20_gflops <= r.median_gflops <= r.q80_gflops
        assert r.kernel
    f = tmp_path / "r.json"
    harness.emit_report(res, "json", f)
    back = harness.load_report(f)
    assert [r.__dict__ for r in back.reports] == [r.__dict__ for r in res.reports]
    c = tmp_path / "r.csv"
    harness.emit_report(res, "csv", c)
    lines = c.read_text().splitlines()
    assert lines[0] == harness.CSV_HEADER and len(lines) == 1 + len(res.reports)


def test_run_benchmark_bf16_tolerance_gate_and_table():
    suite = load_shape_suite("resnet18")[1:5]
    res = harness.run_benchmark(suite, reps=2, warmup=1, dtype=torch.bfloat16, batch=4, min_sample_s=1e-4)
    table = harness.speedup_table(res)
    assert "non-1x1" in table and table["non-1x1"]["shapes"] >= 1


def test_cli_end_to_end_csv(tmp_path):
    out = tmp_path / "o.csv"
    rc = cli.main(["--suite", "squeezenet10", "--variants", "indirect,gemm", "--reps", "2", "--warmup", "1",
                   "--dtype", "bf16", "--batch", "2", "--out", str(out), "--min-sample-ms", "0.1"])
    assert rc == cli.EXIT_OK
    assert out.read_text().splitlines()[0] == harness.CSV_HEADER
    rc = cli.main(["--suite", "squeezenet10", "--variants", "indirect", "--reps", "1", "--out",
                   str(tmp_path / "no" / "dir.csv"), "--min-sample-ms", "0.1", "--batch", "1"])
    assert rc == cli.EXIT_IO
