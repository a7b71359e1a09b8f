"""Randomized parity sweep of the im2col-TMA plans on the GPU: random
geometries (kernel up to 24 taps, strides 1-3, dilations 1-2, asymmetric pads,
channel counts in whole 128-byte blocks, ragged K, small images so that tiles
span rows and images) with im2col_a = 2, single CTAs and CTA pairs:
  bf16: byte-for-byte against the IB-gather kernel (same accumulation order);
  uint8: bit-exact against the gather kernel as well (zero row = zero point,
         TMA zero fill + border-class corrections vs. following the buffer).
    python tools/fuzz_im2col.py [cases] [seed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1907_02129_b200 as icv  # noqa: E402
from paper_1907_02129_b200 import _lib as L  # noqa: E402

DEV = "cuda"


def rand_geom(rng, u8):
    while True:
        r, s = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        if r * s > 24:
            continue
        sy, sx = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        dy, dx = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        pt, pb, pl, pr = (int(v) for v in rng.integers(0, 4, 4))
        h, w = int(rng.integers(3, 21)), int(rng.integers(3, 21))
        if h + pt + pb < (r - 1) * dy + 1 or w + pl + pr < (s - 1) * dx + 1:
            continue
        c = int(rng.choice([128, 256, 384] if u8 else [64, 128, 192, 256]))
        k = int(rng.integers(8, 300))
        n = int(rng.integers(1, 5))
        p = icv.ConvParams(kernel_h=r, kernel_w=s, stride_h=sy, stride_w=sx, dilation_h=dy, dilation_w=dx, pad_top=pt,
                           pad_left=pl, pad_bottom=pb, pad_right=pr, in_channels=c, out_channels=k)
        return p, icv.Shape4(n, h, w, c)


def run(cases: int, seed: int):
    """(kernel runs compared per dtype, mismatches)"""
    rng = np.random.default_rng(seed)
    saved = L.get_tuning("im2col_a"), L.get_tuning("dense_cs")
    L.set_tuning("im2col_a", 2)
    bad = 0
    ran = {"bf16": 0, "u8": 0}
    for i in range(cases):
        u8 = bool(i % 3 == 2)
        p, shape = rand_geom(rng, u8)
        tile = icv.TileConfig(mr=128)
        o = icv.conv_output_shape(p, shape)
        if u8:
            zx, zw = int(rng.integers(0, 256)), int(rng.integers(0, 256))
            xh = rng.integers(0, 256, shape.numel, dtype=np.uint8)
            wh = rng.integers(0, 256, p.out_channels * p.kernel_elems * p.in_channels, dtype=np.uint8)
            bias = rng.integers(-5000, 5000, p.out_channels, dtype=np.int32)
            qp = icv.QuantParams(zx, 0.02, zw, 0.005, 128, 0.1)
            x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV))
            filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
            pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, quant=qp)
            zero = icv.make_zero_row(p.in_channels, dtype=torch.uint8, device=DEV, fill=zx)
            dt = torch.uint8
        else:
            xh = rng.standard_normal(shape.numel, dtype=np.float32)
            wh = rng.standard_normal(p.out_channels * p.kernel_elems * p.in_channels, dtype=np.float32)
            bias = rng.standard_normal(p.out_channels, dtype=np.float32)
            x = icv.NhwcTensor(shape, torch.from_numpy(xh).to(DEV).to(torch.bfloat16))
            filt = icv.FilterTensor(p.out_channels, p.kernel_h, p.kernel_w, p.in_channels, torch.from_numpy(wh).to(DEV))
            pf = icv.pack_filter(filt, torch.from_numpy(bias), p, tile, compute_dtype=torch.bfloat16)
            zero = icv.make_zero_row(p.in_channels, dtype=torch.bfloat16, device=DEV)
            dt = torch.bfloat16
        ib = icv.init_indirection_buffer(x, zero, p, o, tile)
        yg = icv.indirect_conv(x, pf, ib, p, tile, algorithm="gather").numpy().tobytes()
        for cs in (1, 2):
            L.set_tuning("dense_cs", cs)
            name = L.kernel_name(p, shape, dt)
            if "im2col" not in name and "dense" not in name:
                continue          # (not eligible: e.g. a 1x1 stride-1 unpadded layer takes dense boxes)
            y = icv.indirect_conv(x, pf, ib, p, tile).numpy().tobytes()
            ran["u8" if u8 else "bf16"] += 1
            if y != yg:
                bad += 1
                print("MISMATCH", name, p, shape)
    L.set_tuning("im2col_a", saved[0])
    L.set_tuning("dense_cs", saved[1])
    return ran, bad


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    ran, bad = run(cases, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print(f"{cases} geometries, {ran} kernel runs compared with the IB-gather kernel, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
