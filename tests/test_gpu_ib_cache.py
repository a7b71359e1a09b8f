"""IndirectionCache: the paper's reinitialization rules (§2.3,
reference indirect.py:167-212) applied across calls; every buffer it hands
out must equal a freshly built one and give the same convolution."""

import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _fresh(x, zero, p, tile, batch):
    return icv.init_indirection_buffer(x, zero, p, icv.conv_output_shape(p, x.shape), tile, batch=batch)


@pytest.mark.parametrize("per_image", [False, True])
def test_ib_cache_lifecycle(per_image):
    p = make_params(r=3, s=3, pt=1, pl=1, c=16, k=16)
    tile = icv.TileConfig(mr=128)
    zero = icv.make_zero_row(16, dtype=torch.bfloat16, device=DEV)
    filt = icv.filter_fill_random(p, 1, device=DEV)
    pf = icv.pack_filter(filt, None, p, tile, compute_dtype=torch.bfloat16)
    cache = icv.IndirectionCache(p, tile, zero, per_image=per_image)
    shape = icv.Shape4(4, 9, 11, 16)
    x = icv.tensor_fill_random(shape, 0, device=DEV, dtype=torch.bfloat16)

    def conv_ok(inp, batch):
        ib = cache.get(inp, batch)
        ref_ib = _fresh(inp, zero, p, tile, batch)
        if not per_image and ib.batch == batch:   # (a truncated call reuses a larger buffer: outputs compared below)
            assert torch.equal(ib.offsets, ref_ib.offsets)
        y = icv.indirect_conv(inp, pf, ib, p, tile, batch=batch).numpy()
        y_ref = icv.indirect_conv(inp, pf, ref_ib, p, tile, batch=batch).numpy()
        assert (y == y_ref).all()

    conv_ok(x, 2)
    assert cache.stats == icv.CacheStats(builds=1)
    conv_ok(x, 2)                     # same location and batch
    conv_ok(x, 1)                     # logical truncation
    assert cache.stats.hits == 2
    conv_ok(x, 4)                     # growth: only the new part built
    assert cache.stats.growths == 1
    x2 = icv.tensor_fill_random(shape, 5, device=DEV, dtype=torch.bfloat16)
    conv_ok(x2, 4)                    # new location: complete re-initialization
    assert cache.stats.rebinds == 1
    x3 = icv.tensor_fill_random(icv.Shape4(2, 7, 7, 16), 6, device=DEV, dtype=torch.bfloat16)
    conv_ok(x3, 2)                    # new geometry: a new buffer
    assert cache.stats.builds == 2
    with pytest.raises(ValueError):
        cache.get(x3, 3)
