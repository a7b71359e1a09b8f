"""Reference test-facing API that is host-side tensor handling (CPU, no GPU):
``PackedFilter.weights / lane_weights / tile() / lane_view()`` in the
reference's layout (gemm.py:99-124, :153-158) and the single-tile
``indirect_gemm_microkernel`` (indirect.py:215-236), bit-exact with the
oracle's float32 indirect convolution."""

import os
import sys

import numpy as np
import pytest
import torch

import paper_1907_02129_b200 as icv
from conftest import make_params
from oracle import conv as oconv
from oracle import ib as oib

REF_SRC = "/root/reference/pkg/src"


def _pf(params, w_krsc: np.ndarray, nr: int) -> icv.PackedFilter:
    k, rs, c = params.out_channels, params.kernel_elems, params.in_channels
    return icv.PackedFilter(k, rs, c, nr, torch.float32, params, torch.zeros(1, dtype=torch.uint8),
                            torch.zeros(k), krsc=torch.from_numpy(w_krsc.copy()))


def _layout(w: np.ndarray, k: int, rs: int, c: int, nr: int) -> np.ndarray:
    """gemm.py:153-157 restated: (n_tiles, RS*C, nr), zero-padded lanes."""
    nt = -(-k // nr)
    lanes = np.zeros((nt * nr, rs, c), np.float32)
    lanes[:k] = w.reshape(k, rs, c)
    return lanes.reshape(nt, nr, rs, c).transpose(0, 2, 3, 1).reshape(nt, rs * c, nr)


@pytest.mark.parametrize("k,nr", [(6, 8), (16, 8), (7, 3), (1, 1)])
def test_packed_filter_views_follow_reference_layout(k, nr):
    p = make_params(r=3, s=2, c=5, k=k)
    w = np.random.default_rng(k).uniform(-1, 1, k * 6 * 5).astype(np.float32)
    pf = _pf(p, w, nr)
    want = _layout(w, k, 6, 5, nr)
    assert pf.weights.shape == want.shape and np.array_equal(pf.weights.numpy(), want)
    assert np.array_equal(pf.lane_weights.numpy(), want.transpose(1, 0, 2))
    assert np.array_equal(pf.lane_view().numpy(), want.transpose(1, 0, 2))
    for jt in range(pf.n_tiles):
        assert np.array_equal(pf.tile(jt).numpy(), want[jt])
    assert pf.tile(0).data_ptr() == pf.weights.data_ptr()   # a view, as in the reference


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference checkout not present")
def test_packed_filter_views_equal_the_reference_itself():
    sys.path.insert(0, REF_SRC)
    try:
        import convbench as ref
    finally:
        sys.path.remove(REF_SRC)
    rp = ref.ConvParams(kernel_h=3, kernel_w=3, pad_top=1, pad_left=1, pad_bottom=1, pad_right=1,
                        in_channels=4, out_channels=10)
    rf = ref.filter_fill_random(rp, 1)
    rpf = ref.pack_filter(rf, None, rp, ref.TileConfig(mr=4, nr=8))
    p = make_params(r=3, s=3, pt=1, pl=1, c=4, k=10)
    pf = _pf(p, rf.data, 8)
    assert np.array_equal(pf.weights.numpy(), rpf.weights)
    assert np.array_equal(pf.lane_view().numpy(), rpf.lane_view())
    assert np.array_equal(pf.tile(1).numpy(), rpf.tile(1))


@pytest.mark.parametrize("geom", [
    dict(r=3, s=3, pt=1, pl=1, c=4, k=10, n=2, h=5, w=6, mr=4, nr=8),
    dict(r=2, s=3, sy=2, dx=2, pt=1, pl=2, pb=0, pr=1, c=3, k=5, n=1, h=7, w=6, mr=3, nr=2),
])
def test_indirect_gemm_microkernel_bit_exact_with_oracle(geom):
    g = dict(geom)
    n, h, wd, mr, nr = (g.pop(key) for key in ("n", "h", "w", "mr", "nr"))
    p = make_params(**g)
    c, k, rs = p.in_channels, p.out_channels, p.kernel_elems
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, n * h * wd * c).astype(np.float32)
    w = rng.uniform(-1, 1, k * rs * c).astype(np.float32)
    bias = rng.uniform(-1, 1, k).astype(np.float32)
    oh, ow = oib.out_hw(p, h, wd)
    offs = oib.compute_offsets((n, h, wd, c), p, oh, ow, n, mr)
    ref = oconv.indirect_conv_f32(x, np.zeros(c, np.float32), offs, p, w, bias, n, oh, ow)
    pf = _pf(p, w, nr)
    xt, zero = torch.from_numpy(x), torch.zeros(c)
    pixels = n * oh * ow
    for t in range(offs.shape[0]):
        rows = [zero if o < 0 else xt[o:o + c] for e in range(rs) for o in offs[t, e].tolist()]
        for jt in range(pf.n_tiles):
            pb = np.zeros(pf.n_tiles * nr, np.float32)
            pb[:k] = bias
            acc = torch.from_numpy(np.tile(pb.reshape(pf.n_tiles, nr)[jt], (mr, 1)))   # bias init
            out = icv.indirect_gemm_microkernel(rs, c, pf.tile(jt), rows, acc).numpy()
            for m in range(mr):
                px = t * mr + m
                if px >= pixels:
                    break
                cols = slice(jt * nr, min(k, (jt + 1) * nr))
                assert out[m, :cols.stop - cols.start].tobytes() == ref[px, cols].tobytes()
