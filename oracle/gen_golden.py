"""Generate tests/golden/ fixtures by running the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the read-only
reference lives at /root/reference:

    python -m oracle.gen_golden

It imports ``convbench`` from /root/reference/pkg/src (plus the reference's
own test helpers ``oracles.sweep_geometries`` and ``conftest.make_params``)
and records, for every case, the reference's outputs as SHA-256 digests of
their little-endian bytes (plus the full arrays for the smallest cases).
The committed JSON then pins both the numpy oracle (tests/test_oracle_golden.py)
and the CUDA path (tests/test_gpu_parity.py) without the reference being
present.  The GPU box never runs this script.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def params_dict(p) -> dict:
    return {k: int(getattr(p, k)) for k in (
        "kernel_h", "kernel_w", "stride_h", "stride_w", "dilation_h", "dilation_w",
        "pad_top", "pad_left", "pad_bottom", "pad_right", "in_channels", "out_channels")}


def main() -> None:
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    import convbench as cb  # the reference
    from conftest import make_params  # reference test helper
    from oracles import sweep_geometries  # reference test helper
    import torch

    os.makedirs(OUT_DIR, exist_ok=True)

    def build(params, shape, seed, mr, batch=None):
        inp = cb.tensor_fill_random(shape, seed)
        zero = cb.make_zero_row(params.in_channels)
        out_shape = cb.conv_output_shape(params, inp.shape)
        ib = cb.init_indirection_buffer(inp, zero, params, out_shape, cb.TileConfig(mr=mr), batch=batch)
        return inp, zero, out_shape, ib

    # ---- 1. IB known-answer cases (test_indirect.py:40-116 geometries) ----
    kat = []
    kat_geoms = [
        ("pointwise_2x2_mr1", make_params(c=3), cb.Shape4(1, 2, 2, 3), 1, 1),
        ("all_border_1x1_p1", make_params(r=3, s=3, pt=1, pl=1, c=4), cb.Shape4(1, 1, 1, 4), 1, 2),
        ("4x4_mr4", make_params(r=3, s=3, pt=1, pl=1, c=4), cb.Shape4(1, 4, 4, 4), 4, 3),
        ("nonsquare_strided_dilated", make_params(r=3, s=2, sy=2, sx=1, dy=2, dx=1, pt=2, pl=1, c=3),
         cb.Shape4(2, 5, 4, 3), 4, 4),
        ("entry_formula", make_params(r=2, s=3, sy=2, sx=1, pt=1, pl=1, c=2), cb.Shape4(2, 7, 5, 2), 4, 6),
        ("trailing_clamp", make_params(c=2), cb.Shape4(1, 3, 3, 2), 4, 7),
        ("asym_pads", make_params(r=3, s=3, pt=2, pl=0, pb=0, pr=1, sy=1, sx=2, c=5),
         cb.Shape4(2, 6, 7, 5), 3, 8),
    ]
    for mr_extra in (1, 3, 4, 128):
        kat_geoms.append((f"cfg_like_7x7s2p3_mr{mr_extra}",
                          make_params(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3), cb.Shape4(2, 12, 10, 3),
                          mr_extra, 9))
    for name, params, shape, mr, seed in kat_geoms:
        _, _, out_shape, ib = build(params, shape, seed, mr)
        kat.append({"name": name, "params": params_dict(params), "in_shape": list(shape.astuple()),
                    "mr": mr, "batch": shape.n, "out_hw": [out_shape.h, out_shape.w],
                    "offsets_shape": list(ib.offsets.shape),
                    "offsets": ib.offsets.reshape(-1).tolist()})

    # ---- 2. IB sweep digests over the reference sweep grid (oracles.py:145-178) ----
    sweep = []
    for i, params, shape in sweep_geometries(211):
        try:
            out_shape = cb.conv_output_shape(params, shape)
        except cb.InvalidGeometryError:
            continue
        row = {"i": i, "params": params_dict(params), "in_shape": list(shape.astuple()),
               "out_hw": [out_shape.h, out_shape.w], "mr": {}}
        for mr in (1, 3, 4, 128):
            _, _, _, ib = build(params, shape, i, mr)
            row["mr"][str(mr)] = [list(ib.offsets.shape), sha(ib.offsets.astype("<i8"))]
        # batch prefix (logical batch) when N == 2
        if shape.n == 2:
            _, _, _, ib1 = build(params, shape, i, 4, batch=1)
            row["batch1_mr4"] = [list(ib1.offsets.shape), sha(ib1.offsets.astype("<i8"))]
            grown = cb.update_for_batch_growth(ib1, 2)
            row["grown_mr4"] = sha(grown.offsets.astype("<i8"))
        sweep.append(row)

    # ---- 3. f32 conv digests (test_acceptance.py:78-116 operands) ----
    conv = []
    tile = cb.TileConfig(mr=4, nr=8)
    for i, params, shape in sweep_geometries(997):
        try:
            out_shape = cb.conv_output_shape(params, shape)
        except cb.InvalidGeometryError:
            continue
        inp = cb.tensor_fill_random(shape, seed=i)
        filt = cb.filter_fill_random(params, seed=i + 1)
        bias = np.random.default_rng(i + 2).uniform(-1.0, 1.0, params.out_channels).astype(np.float32)
        pf = cb.pack_filter(filt, bias, params, tile)
        ib = cb.init_indirection_buffer(inp, cb.make_zero_row(params.in_channels), params, out_shape, tile)
        out = cb.indirect_conv(inp, pf, ib, params, tile)
        row = {"i": i, "params": params_dict(params), "in_shape": list(shape.astuple()),
               "out_sha": sha(out.data.astype("<f4"))}
        if out.data.size <= 64:
            row["out"] = [float(v) for v in out.data]
        conv.append(row)

    # test_indirect.py conv cases (bias from default_rng(seed+2), filter seed+1)
    conv_kat = []
    for name, params, shape, seed, mr, nr in [
        ("pointwise", make_params(c=5, k=7), cb.Shape4(1, 3, 4, 5), 40, 4, 8),
        ("tails", make_params(r=3, s=3, pt=1, pl=1, c=7, k=9), cb.Shape4(1, 6, 5, 7), 13, 4, 8),
        ("7x7_s2", make_params(r=7, s=7, sy=2, sx=2, pt=3, pl=3, c=3, k=8), cb.Shape4(1, 16, 16, 3), 14, 4, 8),
        ("mr3_nr4", make_params(r=2, s=2, pt=1, pl=1, c=3, k=6), cb.Shape4(1, 4, 5, 3), 20, 3, 4),
        ("big_c_k", make_params(r=3, s=3, pt=1, pl=1, c=64, k=72), cb.Shape4(2, 9, 7, 64), 31, 128, 8),
        ("dilated_asym", make_params(r=3, s=3, dy=2, dx=2, pt=2, pl=2, pb=1, pr=3, sy=2, sx=1, c=16, k=33),
         cb.Shape4(2, 11, 9, 16), 32, 4, 8),
    ]:
        t = cb.TileConfig(mr=mr, nr=nr)
        inp, zero, out_shape, ib = build(params, shape, seed, mr)
        filt = cb.filter_fill_random(params, seed + 1)
        bias = np.random.default_rng(seed + 2).uniform(-1, 1, params.out_channels).astype(np.float32)
        pf = cb.pack_filter(filt, bias, params, t)
        out = cb.indirect_conv(inp, pf, ib, params, t)
        ref = cb.direct_conv(inp, filt, bias, params)
        assert out.data.tobytes() == ref.data.tobytes()
        conv_kat.append({"name": name, "params": params_dict(params), "in_shape": list(shape.astuple()),
                         "seed": seed, "mr": mr, "nr": nr, "out_sha": sha(out.data.astype("<f4"))})

    # ---- 4. cfg1 (BASELINE configs[0]) full f32 output ----
    from paper_1907_02129_b200.workloads import CFG1, CFG2, CFG3A, CFG3B
    w = CFG1
    params = cb.ConvParams(**params_dict(w.params))
    shape = cb.Shape4(*w.in_shape.astuple())
    inp = cb.NhwcTensor(shape, w.input_host())
    filt = cb.FilterTensor(params.out_channels, params.kernel_h, params.kernel_w, params.in_channels,
                           w.filter_host())
    bias = w.bias_host()
    assert np.array_equal(inp.data, cb.tensor_fill_random(shape, 0).data)
    assert np.array_equal(filt.data, cb.filter_fill_random(params, 1).data)
    pf = cb.pack_filter(filt, bias, params, tile)
    out_shape = cb.conv_output_shape(params, shape)
    ib = cb.init_indirection_buffer(inp, cb.make_zero_row(params.in_channels), params, out_shape, tile)
    out = cb.indirect_conv(inp, pf, ib, params, tile)
    cfg1 = {"name": w.name, "out_sha": sha(out.data.astype("<f4")),
            "ib_mr4_sha": sha(ib.offsets.astype("<i8")),
            "out_head": [float(v) for v in out.data[:64]],
            "out_sum": float(out.data.astype(np.float64).sum())}

    # ---- 5. bf16 slices: reference f32 conv on bf16-rounded operands ----
    def bf16(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float32).numpy()

    bf16_cases = []
    for w, n_img in ((CFG2, 1), (CFG3A, 1), (CFG3B, 1)):
        params = cb.ConvParams(**params_dict(w.params))
        shape = cb.Shape4(n_img, w.in_shape.h, w.in_shape.w, w.in_shape.c)
        x = bf16(w.input_host(0, n_img))
        wt = bf16(w.filter_host())
        inp = cb.NhwcTensor(shape, x)
        filt = cb.FilterTensor(params.out_channels, params.kernel_h, params.kernel_w, params.in_channels, wt)
        t = cb.TileConfig(mr=128, nr=8)
        pf = cb.pack_filter(filt, None, params, t)
        out_shape = cb.conv_output_shape(params, shape)
        ib = cb.init_indirection_buffer(inp, cb.make_zero_row(params.in_channels), params, out_shape, t)
        out = cb.indirect_conv(inp, pf, ib, params, t)
        bf16_cases.append({"name": w.name, "images": n_img, "x_bf16_sha": sha(x.astype("<f4")),
                           "w_bf16_sha": sha(wt.astype("<f4")), "ib_mr128_sha": sha(ib.offsets.astype("<i8")),
                           "out_sha": sha(out.data.astype("<f4")),
                           "out_head": [float(v) for v in out.data[:32]],
                           "out_absmax": float(np.abs(out.data).max())})

    doc = {"generator": "oracle/gen_golden.py", "reference": "/root/reference/pkg/src/convbench",
           "digest": "sha256(little-endian bytes)[:32]",
           "ib_kat": kat, "ib_sweep": sweep, "conv_sweep": conv, "conv_kat": conv_kat,
           "cfg1": cfg1, "bf16_slices": bf16_cases}
    path = os.path.join(OUT_DIR, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    print(f"wrote {path}: {len(kat)} KAT, {len(sweep)} IB sweep, {len(conv)} conv sweep, "
          f"{len(conv_kat)} conv KAT, {len(bf16_cases)} bf16 slices")


if __name__ == "__main__":
    main()
