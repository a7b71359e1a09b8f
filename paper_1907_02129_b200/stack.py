"""ResNet-50 convolution stack driven through the indirect-convolution API
(cfg5).

The 53 convolutions of ResNet-50 v1 run chained, each through
``init_indirection_buffer`` / ``pack_filter`` / ``indirect_conv`` exactly as
a caller of the reference operator would (indirect.py:129, gemm.py:135,
indirect.py:239): the IB of every layer is built once against that layer's
persistent input buffer (the paper's persistent-location assumption,
PAPER.md §2.3) and reused on every run.  Conv layers only -- no BN, ReLU or
residual add, as cfg5 specifies; a block's 1x1 expansion output feeds the
next block, its projection reads the block input.  The 3x3/2 p1 max pool
after the stem is the only non-conv op (``icv_maxpool2d``, csrc/pool.cu;
its time is reported separately).

Weights are He-normal (std sqrt(2 / (R*S*C))) with seed = layer index + 1,
the network input N(0, 1) with seed 0, all rounded to bf16.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .gemm import PackedFilter, TileConfig, pack_filter
from .indirect import IndirectionBuffer, indirect_conv, init_indirection_buffer, make_zero_row
from .tensors import ConvParams, FilterTensor, NhwcTensor, Shape4, conv_output_shape
from .workloads import resnet50_layers


def max_pool2d_nhwc(x: NhwcTensor, kernel: int, stride: int, padding: int, out: NhwcTensor | None = None
                    ) -> NhwcTensor:
    """NHWC max pool through the native library (padding taps skipped)."""
    s = x.shape
    oh = (s.h + 2 * padding - kernel) // stride + 1
    ow = (s.w + 2 * padding - kernel) // stride + 1
    shape = Shape4(s.n, oh, ow, s.c)
    if out is None:
        out = NhwcTensor.empty(shape, dtype=x.dtype, device=x.device)
    elif out.shape != shape or out.dtype != x.dtype:
        raise ValueError(f"out must be a {x.dtype} NhwcTensor of shape {shape}")
    L.require_cuda(x.data, "input")
    with torch.cuda.device(x.device):
        L.check(L.lib().icv_maxpool2d(ctypes.byref(L.shape_of(s)), kernel, kernel, stride, stride, padding, padding,
                                      L.TORCH_TO_ICV[x.dtype], L.ptr(x.data), L.ptr(out.data), L.stream_of(x.device)),
                "icv_maxpool2d")
    return out


@dataclass
class StackLayer:
    index: int
    name: str
    params: ConvParams
    input: NhwcTensor
    output: NhwcTensor
    packed: PackedFilter
    ib: IndirectionBuffer
    weights_host: np.ndarray = field(repr=False)     # bf16-rounded KRSC, float32

    @property
    def flops(self) -> int:
        s, p = self.output.shape, self.params
        return 2 * s.n * s.h * s.w * p.out_channels * p.kernel_elems * p.in_channels

    @property
    def compulsory_bytes(self) -> int:
        p = self.params
        return 2 * (self.input.shape.numel + p.out_channels * p.kernel_elems * p.in_channels + self.output.shape.numel)


IMAGE_ELEMS = 224 * 224 * 3


def stack_input_host(lo: int, hi: int) -> np.ndarray:
    """Images [lo, hi) of the network input: the N(0, 1) float32 stream of
    seed 0, image i = elements [i*224*224*3, (i+1)*224*224*3) (so a shard
    holds exactly its slice of the global batch)."""
    x = np.random.default_rng(0).standard_normal(hi * IMAGE_ELEMS, dtype=np.float32)
    return x[lo * IMAGE_ELEMS:]


def stack_weights_host(index: int, params: ConvParams) -> np.ndarray:
    """He-normal KRSC weights of layer ``index`` (seed index + 1), float32."""
    kk = params.kernel_elems * params.in_channels
    wrng = np.random.default_rng(index + 1)
    return wrng.standard_normal(params.out_channels * kk, dtype=np.float32) * np.float32(np.sqrt(2.0 / kk))


class ResNet50Stack:
    """All 53 layers with persistent activations, packed filters and IBs.

    ``images=(lo, hi)`` builds the stack for that slice of the global batch
    (one data-parallel rank's shard); ``replicate``, when
    given, is called with every packed filter right after packing (the
    data-parallel runner broadcasts rank 0's bytes to the other ranks there).
    """

    def __init__(self, batch: int = 256, device="cuda", mr: int = 128, per_image: bool = True,
                 images: tuple[int, int] | None = None, replicate=None):
        self.device = torch.device(device)
        self.tile = TileConfig(mr=mr)
        lo, hi = images if images is not None else (0, batch)
        batch = hi - lo
        self.images = (lo, hi)
        specs = resnet50_layers(batch)
        x0 = stack_input_host(lo, hi)
        self.input = NhwcTensor(Shape4(batch, 224, 224, 3), torch.from_numpy(x0).to(self.device).to(torch.bfloat16))
        self.layers: list[StackLayer] = []
        self.pool_out: NhwcTensor | None = None
        zero_rows: dict[int, torch.Tensor] = {}
        block_in = None
        pending = None          # 1x1b output of the current block -> next block's input
        for idx, (name, shape, params) in enumerate(specs):
            if name == "stem":
                src = self.input
            elif name.endswith("_1x1a"):
                if pending is not None:
                    block_in, pending = pending, None
                src = block_in
            elif name.endswith("_3x3"):
                src = self.layers[-1].output
            elif name.endswith("_1x1b"):
                src = self.layers[-1].output
            else:                                            # projection reads the block input
                src = block_in
            assert src.shape == shape, (name, src.shape, shape)
            out = NhwcTensor.empty(conv_output_shape(params, shape), dtype=torch.bfloat16, device=self.device)
            w = stack_weights_host(idx, params)
            w_dev = torch.from_numpy(w).to(self.device).to(torch.bfloat16)
            filt = FilterTensor(params.out_channels, params.kernel_h, params.kernel_w, params.in_channels, w_dev)
            pf = pack_filter(filt, None, params, self.tile, compute_dtype=torch.bfloat16)
            if replicate is not None:
                replicate(pf)
            c = params.in_channels
            if c not in zero_rows:
                zero_rows[c] = make_zero_row(c, dtype=torch.bfloat16, device=self.device)
            ib = init_indirection_buffer(src, zero_rows[c], params, out.shape, self.tile, per_image=per_image)
            self.layers.append(StackLayer(idx, name, params, src, out, pf, ib, w_dev.float().cpu().numpy()))
            if name == "stem":
                s = out.shape
                self.pool_out = NhwcTensor.empty(Shape4(s.n, (s.h + 1) // 2, (s.w + 1) // 2, s.c),
                                                 dtype=torch.bfloat16, device=self.device)
                block_in = self.pool_out
            elif name.endswith("_1x1b"):
                pending = out
        self.flops = sum(layer.flops for layer in self.layers)

    def maxpool(self) -> None:
        """3x3 / stride 2 / pad 1 max pool of the stem output into pool_out."""
        max_pool2d_nhwc(self.layers[0].output, 3, 2, 1, out=self.pool_out)

    def run_layer(self, layer: StackLayer) -> None:
        indirect_conv(layer.input, layer.packed, layer.ib, layer.params, self.tile, out=layer.output)

    def run(self, events: list | None = None) -> None:
        """One pass of the whole stack; with ``events`` (a list of 55 CUDA
        events) records a timestamp before each layer, after the pool and at
        the end."""
        for i, layer in enumerate(self.layers):
            if events is not None:
                events[i + (1 if i > 0 else 0)].record()
            self.run_layer(layer)
            if i == 0:
                if events is not None:
                    events[1].record()
                self.maxpool()
        if events is not None:
            events[-1].record()

    def graphed(self):
        """The whole pass (53 convolutions + max pool) captured once as a CUDA
        graph; returns a callable that replays it on the current stream.  The
        kernels' programmatic-dependent-launch edges are kept by the capture,
        and no host work remains per pass."""
        g = torch.cuda.CUDAGraph()
        self.run()                              # (every kernel attribute / tensor map set up once)
        torch.cuda.synchronize(self.device)
        side = torch.cuda.Stream(self.device)
        n0 = L.launch_count()
        with torch.cuda.stream(side):
            g.capture_begin()
            self.run()
            g.capture_end()
        self.graph_launches = L.launch_count() - n0   # libicv kernels in one replay
        torch.cuda.synchronize(self.device)
        self._graph = g                         # keep it alive with the stack
        return g.replay

    def timed_run(self) -> tuple[float, float, list[float]]:
        """(total ms, max-pool ms, per-layer conv ms) of one pass, CUDA events."""
        n = len(self.layers)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 2)]
        self.run(ev)
        torch.cuda.synchronize()
        # ev[0] stem start, ev[1] stem end / pool start, ev[2] pool end / layer 1 start, ...
        per = [ev[0].elapsed_time(ev[1])]
        pool = ev[1].elapsed_time(ev[2])
        for i in range(1, n):
            per.append(ev[i + 1].elapsed_time(ev[i + 2]))
        return ev[0].elapsed_time(ev[-1]), pool, per
