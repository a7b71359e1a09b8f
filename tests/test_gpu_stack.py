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
