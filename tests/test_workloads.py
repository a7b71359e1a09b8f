"""BASELINE.json workload definitions (synthetic inputs; no dataset is used)
against the analytic numbers in SURVEY.md §0 / Appendix B.  CPU only."""

import numpy as np

from paper_1907_02129_b200.workloads import CFG1, CFG2, CFG3A, CFG3B, CFG4, resnet50_layers


def test_flops_and_compulsory_bytes():
    # GFLOP and compulsory MB
    assert round(CFG1.flops / 1e9, 3) == 0.231
    assert round(CFG2.flops / 1e9, 3) == 14.798
    assert round(CFG3A.flops / 1e9, 3) == 7.553
    assert round(CFG3B.flops / 1e9, 3) == 77.309
    assert round(CFG4.flops / 1e9, 3) == 29.595
    assert round(CFG2.compulsory_bytes / 1e6, 2) == 25.99
    assert round(CFG3A.compulsory_bytes / 1e6, 2) == 61.03
    assert round(CFG4.compulsory_bytes / 1e6, 2) == 32.70


def test_output_shapes():
    assert CFG2.out_hw == (28, 28)
    assert CFG3A.out_hw == (112, 112)
    assert CFG3B.out_hw == (64, 64)
    assert CFG4.out_hw == (14, 14)


def test_generators_are_deterministic_and_shard_consistent():
    x = CFG2.input_host()
    assert x.dtype == np.float32 and x.size == 64 * 28 * 28 * 128
    per = 28 * 28 * 128
    assert np.array_equal(CFG2.input_host(3, 5), x[3 * per:5 * per])
    w = CFG2.filter_host()
    assert abs(float(w.std()) - np.sqrt(2.0 / 1152)) < 2e-3           # He-normal
    b = CFG4.bias_host()
    assert b.dtype == np.int32 and b.min() >= -1000 and b.max() <= 1000
    u = CFG4.input_host(0, 1)
    assert u.dtype == np.uint8
    assert np.array_equal(CFG1.bias_host(), np.random.default_rng(2).uniform(-1, 1, 64).astype(np.float32))


def test_resnet50_stack():
    layers = resnet50_layers(256)
    assert len(layers) == 53
    gflop = sum(2 * s.n * ((s.h + p.pad_top + p.pad_bottom - p.kernel_h) // p.stride_h + 1)
                * ((s.w + p.pad_left + p.pad_right - p.kernel_w) // p.stride_w + 1)
                * p.out_channels * p.kernel_elems * p.in_channels for _, s, p in layers) / 1e9
    assert round(gflop, 1) == 2092.6
    params = sum(p.out_channels * p.kernel_elems * p.in_channels for _, _, p in layers)
    assert params == 23454912
