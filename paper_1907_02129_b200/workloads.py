"""Seeded synthetic inputs for the BASELINE.json configurations.

No dataset or checkpoint is involved anywhere in BASELINE.json: every config
is synthetic.  Seeds follow the reference harness convention
(/root/reference/pkg/src/convbench/bench.py:215-219): input seed s, filter
s+1, bias s+2, with s = 0.  Values are generated on the host with numpy's
``default_rng`` (so any slice of the batch is reproducible independently of
how the batch is later sharded across GPUs) and uploaded once.

  cfg1  f32   1x56x56x64 -> 64, 3x3 s1 p1, U(-1,1) input/filter/bias
  cfg2  bf16  64x28x28x128 -> 128, 3x3 s1 p1, N(0,1) input, He-normal filter, zero bias
  cfg3a bf16  32x224x224x3 -> 64, 7x7 s2 p3 (channel-poor stem)
  cfg3b bf16  16x64x64x256 -> 256, 3x3 d2 p2
  cfg4  u8    128x28x28x256 -> 256, 3x3 s2 p1, QNNPACK asymmetric quantization
  cfg5  bf16  ResNet-50 v1 conv stack, N=256 (53 convs + maxpool after the stem)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .tensors import ConvParams, Shape4


@dataclass(frozen=True)
class QuantSpec:
    """Asymmetric uint8 quantization of one convolution (QNNPACK style)."""

    input_zero_point: int = 128
    input_scale: float = 0.02
    kernel_zero_point: int = 127
    kernel_scale: float = 0.005
    output_zero_point: int = 128
    output_scale: float = 0.1
    output_min: int = 0
    output_max: int = 255


@dataclass(frozen=True)
class ConvWorkload:
    name: str
    dtype: str                      # "f32" | "bf16" | "u8"
    in_shape: Shape4
    params: ConvParams
    input_dist: str = "normal"      # "uniform" | "normal" | "u8"
    bias: str = "none"              # "none" | "uniform" | "int32"
    seed: int = 0
    quant: QuantSpec | None = None
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def out_hw(self) -> tuple[int, int]:
        p, s = self.params, self.in_shape
        oh = (s.h + p.pad_top + p.pad_bottom - p.dilation_h * (p.kernel_h - 1) - 1) // p.stride_h + 1
        ow = (s.w + p.pad_left + p.pad_right - p.dilation_w * (p.kernel_w - 1) - 1) // p.stride_w + 1
        return oh, ow

    @property
    def flops(self) -> int:
        """2*N*Ho*Wo*K*R*S*C (BASELINE metric; analysis.py:47-53)."""
        oh, ow = self.out_hw
        p = self.params
        return 2 * self.in_shape.n * oh * ow * p.out_channels * p.kernel_elems * p.in_channels

    def elem_bytes(self) -> tuple[int, int, int]:
        """(input, weight, output) element sizes."""
        return {"f32": (4, 4, 4), "bf16": (2, 2, 2), "u8": (1, 1, 1)}[self.dtype]

    @property
    def compulsory_bytes(self) -> int:
        """Algorithmic HBM bytes: input + filter + output + 4-byte bias per
        output channel.  Indirection-buffer bytes are
        overhead and are not counted here."""
        ei, ew, eo = self.elem_bytes()
        oh, ow = self.out_hw
        p, s = self.params, self.in_shape
        return (s.numel * ei + p.out_channels * p.kernel_elems * p.in_channels * ew
                + s.n * oh * ow * p.out_channels * eo + 4 * p.out_channels)

    def with_batch(self, n: int) -> "ConvWorkload":
        s = self.in_shape
        return ConvWorkload(self.name, self.dtype, Shape4(n, s.h, s.w, s.c), self.params,
                            self.input_dist, self.bias, self.seed, self.quant, self.note, self.extra)

    # -- host-side generators (numpy; identical values for any sharding) --
    def input_host(self, n_lo: int = 0, n_hi: int | None = None) -> np.ndarray:
        """Flat host input for images [n_lo, n_hi): float32 (bf16 configs are
        rounded to bf16 on upload) or uint8."""
        s = self.in_shape
        n_hi = s.n if n_hi is None else n_hi
        per = s.h * s.w * s.c
        rng = np.random.default_rng(self.seed)
        if self.input_dist == "uniform":
            full = rng.uniform(-1.0, 1.0, s.numel).astype(np.float32)
        elif self.input_dist == "normal":
            full = rng.standard_normal(s.numel, dtype=np.float32)
        elif self.input_dist == "u8":
            full = rng.integers(0, 256, s.numel, dtype=np.uint8)
        else:
            raise ValueError(self.input_dist)
        return full[n_lo * per:n_hi * per]

    def filter_host(self) -> np.ndarray:
        """Flat KRSC filter."""
        p = self.params
        count = p.out_channels * p.kernel_elems * p.in_channels
        rng = np.random.default_rng(self.seed + 1 + self.extra.get("filter_seed_offset", 0))
        if self.input_dist == "uniform":
            return rng.uniform(-1.0, 1.0, count).astype(np.float32)
        if self.input_dist == "u8":
            return rng.integers(0, 256, count, dtype=np.uint8)
        std = math.sqrt(2.0 / (p.kernel_elems * p.in_channels))   # He-normal
        return (rng.standard_normal(count, dtype=np.float32) * np.float32(std)).astype(np.float32)

    def bias_host(self) -> np.ndarray | None:
        k = self.params.out_channels
        rng = np.random.default_rng(self.seed + 2)
        if self.bias == "none":
            return None
        if self.bias == "uniform":
            return rng.uniform(-1.0, 1.0, k).astype(np.float32)
        if self.bias == "int32":
            return rng.integers(-1000, 1000, k, dtype=np.int32, endpoint=True)
        raise ValueError(self.bias)


def _p(r, s, stride=1, pad=0, dil=1, c=1, k=1) -> ConvParams:
    return ConvParams(kernel_h=r, kernel_w=s, stride_h=stride, stride_w=stride,
                      dilation_h=dil, dilation_w=dil, pad_top=pad, pad_left=pad,
                      pad_bottom=pad, pad_right=pad, in_channels=c, out_channels=k)


CFG1 = ConvWorkload("cfg1_f32_56x56x64_3x3", "f32", Shape4(1, 56, 56, 64), _p(3, 3, 1, 1, 1, 64, 64),
                    input_dist="uniform", bias="uniform",
                    note="fp32 parity/plumbing case; bit-exact vs the reference")
CFG2 = ConvWorkload("cfg2_bf16_64x28x28x128_3x3", "bf16", Shape4(64, 28, 28, 128),
                    _p(3, 3, 1, 1, 1, 128, 128), note="headline bench workload")
CFG3A = ConvWorkload("cfg3a_bf16_stem_32x224x224x3_7x7s2", "bf16", Shape4(32, 224, 224, 3),
                     _p(7, 7, 2, 3, 1, 3, 64), note="channel-poor, HBM-bound")
CFG3B = ConvWorkload("cfg3b_bf16_16x64x64x256_3x3d2", "bf16", Shape4(16, 64, 64, 256),
                     _p(3, 3, 1, 2, 2, 256, 256))
CFG4 = ConvWorkload("cfg4_u8_128x28x28x256_3x3s2", "u8", Shape4(128, 28, 28, 256),
                    _p(3, 3, 2, 1, 1, 256, 256), input_dist="u8", bias="int32", quant=QuantSpec())

CONFIGS = {"cfg1": CFG1, "cfg2": CFG2, "cfg3a": CFG3A, "cfg3b": CFG3B, "cfg4": CFG4}


def resnet50_layers(batch: int = 256) -> list[tuple[str, Shape4, ConvParams]]:
    """The 53 convolutions of ResNet-50 v1 (torchvision placement: stride on
    the 3x3 of the first block of stages 2-4 and on its projection),
    SURVEY.md Appendix B.  Input shapes assume the 3x3/2 p1 maxpool after the
    stem (112 -> 56)."""
    layers = [("stem", Shape4(batch, 224, 224, 3), _p(7, 7, 2, 3, 1, 3, 64))]
    hw, cin = 56, 64
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)], start=1):
        cout = width * 4
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 1) else 1
            pre = f"s{stage}b{b + 1}"
            layers.append((f"{pre}_1x1a", Shape4(batch, hw, hw, cin), _p(1, 1, 1, 0, 1, cin, width)))
            layers.append((f"{pre}_3x3", Shape4(batch, hw, hw, width), _p(3, 3, stride, 1, 1, width, width)))
            ohw = hw // stride
            layers.append((f"{pre}_1x1b", Shape4(batch, ohw, ohw, width), _p(1, 1, 1, 0, 1, width, cout)))
            if b == 0:
                layers.append((f"{pre}_proj", Shape4(batch, hw, hw, cin), _p(1, 1, stride, 0, 1, cin, cout)))
            hw, cin = ohw, cout
    return layers
