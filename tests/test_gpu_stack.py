"""cfg5: the ResNet-50 conv stack run chained through the indirect API, every
layer checked against the oracle on its actual bf16 input (SURVEY.md §8(d):
parity per layer on a subset of images -- here the first and last image of a
3-image batch, sampled output pixels)."""

import numpy as np
import pytest
import torch

from helpers import assert_bf16_close
from oracle import conv as oconv
from oracle import ib as oib

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def test_resnet50_stack_every_layer_matches_oracle():
    from paper_1907_02129_b200 import _lib as L
    from paper_1907_02129_b200.stack import ResNet50Stack

    stack = ResNet50Stack(batch=3, device=DEV)
    assert len(stack.layers) == 53
    stack.run()
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    for layer in stack.layers:
        p, s = layer.params, layer.input.shape
        o = layer.output.shape
        assert L.kernel_name(p, s, torch.bfloat16).startswith("icv_igemm_")   # tcgen05 path for every layer
        x_all = layer.input.numpy().reshape(s.n, -1)
        y_all = layer.output.numpy().reshape(o.n, o.h * o.w, o.c)
        offs = oib.compute_offsets((1, s.h, s.w, s.c), p, o.h, o.w, 1, 128)
        for n in (0, s.n - 1):
            idx = np.unique(np.concatenate([[0, o.h * o.w - 1], rng.integers(0, o.h * o.w, 192)]))
            ref = oconv.indirect_conv_f32(x_all[n], np.zeros(s.c, np.float32), offs, p, layer.weights_host, None,
                                          1, o.h, o.w, pixel_index=idx)
            assert_bf16_close(y_all[n][idx], ref, what=f"{layer.name} image {n}")


def test_resnet50_stack_maxpool_matches_torch():
    from paper_1907_02129_b200.stack import ResNet50Stack

    stack = ResNet50Stack(batch=2, device=DEV)
    stack.run()
    s = stack.layers[0].output.shape
    x = stack.layers[0].output.data.view(s.n, s.h, s.w, s.c).float().permute(0, 3, 1, 2)
    ref = torch.nn.functional.max_pool2d(x, 3, 2, 1).permute(0, 2, 3, 1).reshape(-1)
    assert torch.equal(stack.pool_out.data.float(), ref)


def test_graph_replay_with_pdl_equals_eager_calls(tune):
    """The bench's timed cfg5 step replays the pass as one CUDA graph whose
    kernels use programmatic dependent launch: every layer's output must be
    byte-identical to eager calls without PDL (a missing griddepcontrol.wait
    would let a layer read its input before the previous layer finished)."""
    from paper_1907_02129_b200.stack import ResNet50Stack

    stack = ResNet50Stack(batch=16, device=DEV)
    tune(pdl=0)
    stack.run()
    torch.cuda.synchronize()
    eager = [l.output.data.clone() for l in stack.layers]
    for l in stack.layers:
        l.output.data.zero_()
    tune(pdl=1)
    replay = stack.graphed()
    for l in stack.layers:
        l.output.data.zero_()
    for _ in range(3):
        replay()
    torch.cuda.synchronize()
    for l, ref in zip(stack.layers, eager):
        assert torch.equal(l.output.data, ref), l.name
    assert stack.graph_launches >= 53


def test_sharded_stack_equals_full_batch():
    """Two shards of the cfg5 stack (images [0, 4) and [4, 8), as two ranks
    would build them) produce the full-batch stack's final activation."""
    from paper_1907_02129_b200.stack import ResNet50Stack

    full = ResNet50Stack(batch=8, device=DEV)
    full.run()
    parts = []
    for lo, hi in ((0, 4), (4, 8)):
        s = ResNet50Stack(device=DEV, images=(lo, hi))
        s.run()
        parts.append(s.layers[-1].output.data.clone())
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts), full.layers[-1].output.data)
