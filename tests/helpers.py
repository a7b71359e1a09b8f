"""Shared helpers for the parity tests (device path vs the numpy oracle)."""

from __future__ import annotations

import hashlib

import numpy as np

REL_TOL_BF16 = 1e-2   # BASELINE.json configs[1]: "rel 1e-2 against the fp32 oracle"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def fill_uniform(numel: int, seed: int) -> np.ndarray:
    """tensors.py:219-223 / :226-234 (identical numpy stream)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, numel).astype(np.float32)


def assert_bf16_close(got: np.ndarray, ref: np.ndarray, rel: float = REL_TOL_BF16, what: str = "") -> dict:
    """The bf16 tolerance of this repo: normwise
    max|got - ref| / max|ref| <= rel AND elementwise
    |got - ref| <= rel*|ref| + rel*rms(ref)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    err = np.abs(got - ref)
    scale = np.abs(ref).max() if ref.size else 1.0
    rms = float(np.sqrt(np.mean(ref * ref))) if ref.size else 1.0
    normwise = float(err.max() / scale) if ref.size else 0.0
    bad = err > rel * np.abs(ref) + rel * rms
    assert normwise <= rel, f"{what}: normwise rel error {normwise:.3e} > {rel}"
    assert not bad.any(), f"{what}: {int(bad.sum())} elements outside rtol={rel}, atol={rel}*rms"
    return {"normwise": normwise, "max_abs": float(err.max()) if ref.size else 0.0}
