"""Known-answer tests for the uint8 oracle (oracle/quant.py).

The reference has no quantized path (tensors.py:107-108), so this oracle's
parity is unpinned against the reference; these tests pin its integer
semantics independently.  CPU only.
"""

import itertools

import numpy as np
import pytest

from conftest import make_params
from oracle import ib as oib
from oracle import quant as oq


def test_requant_params_cfg4_worked_numbers():
    # sx=0.02, sw=0.005, so=0.1 -> M0=1,099,511,562, shift=9
    assert oq.requant_params(0.02, 0.005, 0.1) == (1099511562, 9)


def test_requant_params_rejects_out_of_range():
    with pytest.raises(ValueError):
        oq.requant_params(1.0, 1.0, 0.5)


def test_srdhm_known_answers():
    i32min = -(1 << 31)
    assert oq.srdhm(np.array([i32min]), i32min)[0] == (1 << 31) - 1
    assert oq.srdhm(np.array([1 << 30]), 1 << 30)[0] == 1 << 29
    assert oq.srdhm(np.array([-(1 << 30)]), 1 << 30)[0] == -(1 << 29)
    # 3 * 2**30 / 2**31 = +-1.5: gemmlowp's nudge + truncating division rounds
    # exact ties toward +inf (1.5 -> 2, -1.5 -> -1)
    assert oq.srdhm(np.array([3]), 1 << 30)[0] == 2
    assert oq.srdhm(np.array([-3]), 1 << 30)[0] == -1
    assert oq.srdhm(np.array([-5]), 1 << 30)[0] == -2
    assert oq.srdhm(np.array([1]), 1 << 30)[0] == 1
    assert oq.srdhm(np.array([-1]), 1 << 30)[0] == 0


def test_rounding_divide_by_pot_known_answers():
    cases = [(5, 1, 3), (-5, 1, -3), (4, 1, 2), (-4, 1, -2), (3, 1, 2), (-3, 1, -2),
             (7, 2, 2), (-7, 2, -2), (6, 2, 2), (-6, 2, -2), (5, 2, 1), (-5, 2, -1), (0, 5, 0)]
    for x, e, want in cases:
        assert oq.rounding_divide_by_pot(np.array([x]), e)[0] == want, (x, e)


def _brute_acc(x4, w4, bias, p, zx, zw):
    """Literal loop nest: padding taps skipped, which must equal the zero row
    filled with zx (contributes (zx - zx)(w - zw) = 0)."""
    n, h, w, c = x4.shape
    oh, ow = oib.out_hw(p, h, w)
    k = p.out_channels
    acc = np.zeros((n, oh, ow, k), np.int64)
    for b, oy, ox, kk in itertools.product(range(n), range(oh), range(ow), range(k)):
        a = int(bias[kk]) if bias is not None else 0
        for ky, kx in itertools.product(range(p.kernel_h), range(p.kernel_w)):
            iy = oy * p.stride_h + ky * p.dilation_h - p.pad_top
            ix = ox * p.stride_w + kx * p.dilation_w - p.pad_left
            if 0 <= iy < h and 0 <= ix < w:
                for ci in range(c):
                    a += (int(x4[b, iy, ix, ci]) - zx) * (int(w4[kk, ky, kx, ci]) - zw)
        acc[b, oy, ox, kk] = a
    return acc.reshape(-1, k)


@pytest.mark.parametrize("mr", [1, 4, 128])
def test_u8_acc_matches_loop_nest(mr):
    rng = np.random.default_rng(5)
    p = make_params(r=3, s=3, sy=2, sx=1, dy=1, dx=2, pt=1, pl=2, pb=2, pr=0, c=5, k=7)
    n, h, w = 2, 6, 7
    x = rng.integers(0, 256, n * h * w * p.in_channels, dtype=np.uint8)
    wt = rng.integers(0, 256, p.out_channels * 9 * p.in_channels, dtype=np.uint8)
    bias = rng.integers(-1000, 1000, p.out_channels, dtype=np.int32, endpoint=True)
    oh, ow = oib.out_hw(p, h, w)
    offs = oib.compute_offsets((n, h, w, p.in_channels), p, oh, ow, n, mr)
    zero = np.full(p.in_channels, 128, np.uint8)
    acc = oq.indirect_conv_acc(x, zero, offs, p, wt, bias, n, oh, ow, 128, 127)
    want = _brute_acc(x.reshape(n, h, w, -1), wt.reshape(p.out_channels, 3, 3, -1), bias, p, 128, 127)
    assert np.array_equal(acc, want)


def test_u8_output_clamps_and_zero_point():
    p = make_params(c=1, k=1)
    x = np.array([0, 128, 255], np.uint8)
    offs = oib.compute_offsets((1, 1, 3, 1), p, 1, 3, 1, 1)
    zero = np.full(1, 128, np.uint8)
    # w - zw = 255 - 127 = 128; acc = (x - 128) * 128 -> -16384, 0, 16256
    y = oq.indirect_conv_u8(x, zero, offs, p, np.array([255], np.uint8), None, 1, 1, 3,
                            128, 0.02, 127, 0.005, 128, 0.1)
    # real scale 0.001 -> -16.384 -> -16 + 128 = 112; 0 -> 128; 16.256 -> 16 + 128 = 144
    assert y.reshape(-1).tolist() == [112, 128, 144]


def test_u8_cross_check_torch_qnnpack():
    """Third-party cross-check (not under /root/reference): torch's CPU
    quantized conv.  Its requantization rounding may differ on near-ties,
    so only the mismatch rate is bounded, not bit-equality."""
    torch = pytest.importorskip("torch")
    if "qnnpack" not in torch.backends.quantized.supported_engines:
        pytest.skip("qnnpack engine unavailable")
    rng = np.random.default_rng(11)
    n, h, w, c, k = 2, 9, 9, 16, 24
    p = make_params(r=3, s=3, sy=2, sx=2, pt=1, pl=1, c=c, k=k)
    x = rng.integers(0, 256, n * h * w * c, dtype=np.uint8)
    wt = rng.integers(1, 255, k * 9 * c, dtype=np.uint8)  # int8 recast needs w - 127 in [-127, 127]
    bias = rng.integers(-1000, 1000, k, dtype=np.int32, endpoint=True)
    oh, ow = oib.out_hw(p, h, w)
    offs = oib.compute_offsets((n, h, w, c), p, oh, ow, n, 4)
    ours = oq.indirect_conv_u8(x, np.full(c, 128, np.uint8), offs, p, wt, bias, n, oh, ow,
                               128, 0.02, 127, 0.005, 128, 0.1).reshape(n, oh, ow, k)
    prev = torch.backends.quantized.engine
    try:
        torch.backends.quantized.engine = "qnnpack"
        xq = torch.quantize_per_tensor(
            torch.from_numpy((x.reshape(n, h, w, c).astype(np.float32) - 128) * np.float32(0.02)).permute(0, 3, 1, 2),
            0.02, 128, torch.quint8)
        wf = (wt.reshape(k, 3, 3, c).astype(np.float32) - 127) * np.float32(0.005)
        wq = torch.quantize_per_tensor(torch.from_numpy(wf).permute(0, 3, 1, 2).contiguous(), 0.005, 0, torch.qint8)
        conv = torch.ao.nn.quantized.Conv2d(c, k, 3, stride=2, padding=1)
        conv.set_weight_bias(wq, torch.from_numpy(bias.astype(np.float32) * np.float32(0.02 * 0.005)))
        conv.scale, conv.zero_point = 0.1, 128
        theirs = conv(xq).int_repr().permute(0, 2, 3, 1).numpy()
    finally:
        torch.backends.quantized.engine = prev
    diff = np.abs(ours.astype(np.int32) - theirs.astype(np.int32))
    assert diff.max() <= 1
    assert (diff != 0).mean() < 0.02
