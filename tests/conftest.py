"""Shared test fixtures.

Markers: ``gpu`` = needs a CUDA device (B200) and the built libicv.so;
everything else runs on the CPU (oracle vs golden fixtures, host logic,
C-ABI symbol table, multi-process gloo tests).
"""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and the built libicv.so")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


class P:
    """Minimal ConvParams stand-in built from a golden-fixture dict."""

    def __init__(self, d):
        self.__dict__.update(d)
        self.kernel_elems = self.kernel_h * self.kernel_w


def make_params(r=1, s=1, sy=1, sx=1, dy=1, dx=1, pt=0, pl=0, pb=None, pr=None, c=1, k=1):
    """Compact ConvParams builder mirroring the reference's tests/conftest.py:20-30."""
    from paper_1907_02129_b200.tensors import ConvParams

    return ConvParams(kernel_h=r, kernel_w=s, stride_h=sy, stride_w=sx, dilation_h=dy, dilation_w=dx,
                      pad_top=pt, pad_left=pl, pad_bottom=pt if pb is None else pb,
                      pad_right=pl if pr is None else pr, in_channels=c, out_channels=k)


@pytest.fixture
def tune():
    """Set native plan knobs for one test (icv_set_tuning); restored afterwards."""
    from paper_1907_02129_b200 import _lib as L

    saved = {}

    def set_(**knobs):
        for k, v in knobs.items():
            if k not in saved:
                saved[k] = L.get_tuning(k)
            L.set_tuning(k, v)

    yield set_
    for k, v in saved.items():
        L.set_tuning(k, v)
