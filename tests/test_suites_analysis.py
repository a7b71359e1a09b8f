"""Shape suites and analytical cost models (CPU): the generated builtin
suites equal the reference's data files shape for shape, the file loader
keeps the reference's schema and errors, and the cost models follow
analysis.py's formulas (checked against the reference itself when the
checkout is present, and against hand-computed values always)."""

import json
import os
import sys

import pytest

import paper_1907_02129_b200 as icv
from paper_1907_02129_b200 import analysis as A
from paper_1907_02129_b200 import suites as S
from paper_1907_02129_b200.errors import SuiteParseError

REF_SRC = "/root/reference/pkg/src"
REF_DATA = os.path.join(REF_SRC, "convbench", "data")


def _t(sh):
    return (sh.n, sh.h, sh.w, sh.c)


def _key(spec):
    p = spec.params
    return (spec.name, _t(spec.input_shape), p.kernel_h, p.kernel_w, p.stride_h, p.stride_w, p.dilation_h,
            p.dilation_w, p.pad_top, p.pad_left, p.pad_bottom, p.pad_right, p.out_channels)


@pytest.mark.skipif(not os.path.isdir(REF_DATA), reason="reference checkout not present")
@pytest.mark.parametrize("name", ["resnet18", "squeezenet10"])
def test_generated_builtin_suites_equal_reference_files(name):
    ours = S.load_shape_suite(name)
    theirs = S.load_shape_suite(os.path.join(REF_DATA, f"{name}.json"))
    assert [_key(s) for s in ours] == [_key(s) for s in theirs]
    assert all(s.model == name for s in ours)


def test_builtin_suite_sizes_and_census():
    rn18 = S.load_shape_suite("resnet18")
    assert len(rn18) == 11 and rn18[0].name == "rn18_conv1_7x7_s2"
    assert S.census(rn18) == {"7x7/2": 1, "3x3/2": 3, "3x3/1": 4, "1x1/2": 3, "1x1/1": 0, "other": 0}
    sq = S.load_shape_suite("squeezenet10")
    assert len(sq) == 22 and sq[-1].params.out_channels == 1000
    rn50 = S.load_shape_suite("resnet50", batch=8)
    assert all(s.input_shape.n == 8 for s in rn50)
    assert len({(_key(s)[1:]) for s in rn50}) == len(rn50)


def test_suite_file_roundtrip_and_errors(tmp_path):
    doc = S.builtin_suite_document("resnet18")
    f = tmp_path / "s.json"
    f.write_text(json.dumps(doc))
    assert [_key(s) for s in S.load_shape_suite(str(f))] == [_key(s) for s in S.load_shape_suite("resnet18")]
    bad = dict(doc, version=2)
    f.write_text(json.dumps(bad))
    with pytest.raises(SuiteParseError, match="version"):
        S.load_shape_suite(str(f))
    dup = dict(doc, shapes=doc["shapes"][:1] * 2)
    f.write_text(json.dumps(dup))
    with pytest.raises(SuiteParseError, match="duplicate"):
        S.load_shape_suite(str(f))
    f.write_text("{not json")
    with pytest.raises(SuiteParseError, match="invalid JSON"):
        S.load_shape_suite(str(f))
    with pytest.raises(SuiteParseError, match="cannot read"):
        S.load_shape_suite(str(tmp_path / "missing.json"))
    geom = dict(doc, shapes=[dict(doc["shapes"][0], kernel=[300, 300])])
    f.write_text(json.dumps(geom))
    with pytest.raises(SuiteParseError):
        S.load_shape_suite(str(f))


def test_cost_models_hand_values():
    p = icv.ConvParams(3, 3, pad_top=1, pad_left=1, pad_bottom=1, pad_right=1, in_channels=128, out_channels=128)
    s = icv.Shape4(64, 28, 28, 128)
    o = icv.conv_output_shape(p, s)
    macs, flops = A.flop_count(p, o)
    assert flops == 14_797_504_512 and macs * 2 == flops                    # cfg2: 14.798 GFLOP
    assert A.im2col_overhead(p, o) == 2 * 64 * 128 * 28 * 28 * 9
    assert A.roofline_speedup(4.0, 8) == 2.0
    with pytest.raises(ValueError):
        A.roofline_speedup(-1, 8)
    fp = A.footprint_compare(p, s, icv.TileConfig(mr=128), ref_size=8, elem_bytes=2)
    assert fp.patch_matrix_bytes == 115_605_504                            # 115.6 MB
    assert fp.indirection_bytes == 451_584 * 8
    lam = A.b200_lambda("bf16", {"hbm_gbs": 6450.3, "bf16_tflops": 1667.6})
    assert 515 < lam < 520
    cr = A.cost_report(p, s, icv.TileConfig(mr=128), lam=lam, elem_bytes=2)
    assert cr.speedup_predicted == pytest.approx(1 + 2 * lam / 128)
    d = A.device_footprint(p, s)
    assert d["ib_entries"] == 7 * 9 * 128 and d["patch_over_ib"] > 100


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference checkout not present")
def test_cost_report_equals_reference():
    sys.path.insert(0, REF_SRC)
    try:
        import convbench as ref
    finally:
        sys.path.remove(REF_SRC)
    for spec in S.load_shape_suite("squeezenet10")[:6] + S.load_shape_suite("resnet18"):
        p = spec.params
        rp = ref.ConvParams(**{f: getattr(p, f) for f in ("kernel_h", "kernel_w", "stride_h", "stride_w",
                                                           "dilation_h", "dilation_w", "pad_top", "pad_left",
                                                           "pad_bottom", "pad_right", "in_channels", "out_channels")})
        rs = ref.Shape4(*_t(spec.input_shape))
        for mr, ref_size, lam in ((4, 8, 0.0), (128, 4, 3.5)):
            a = A.cost_report(p, spec.input_shape, icv.TileConfig(mr=mr), ref_size, lam)
            b = ref.cost_report(rp, rs, ref.TileConfig(mr=mr), ref_size, lam)
            assert a.__dict__ == b.__dict__, spec.name
