"""Seeded matrix recipes shared by the golden generator and the tests.

Pure numpy, no reference import: the GPU box regenerates the same inputs
from these recipes and checks them against digests that
``make_golden.py`` recorded from the reference here.

Recipes restate the shapes of the reference's own test inputs:
* ``low_entropy``   — conftest ``random_low_entropy_matrix`` (tests/conftest.py:47-55)
* ``criterion3``    — integer alphabets, m,n <= 500, K <= 128 (tests/test_acceptance.py:108-126)
* ``quantized``     — real (float64, not fp32-representable) alphabets on a uniform grid
                      (tests/test_acceptance.py:128-138 shape; own quantiser)
* ``nonzero_mode``  — quantised uniform(0.25, 2) so the mode is non-zero
                      (tests/test_acceptance.py:238-255 shape)
"""

from __future__ import annotations

import numpy as np


def low_entropy(seed: int, max_mn: int = 40, max_k: int = 8):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, max_mn))
    n = int(rng.integers(1, max_mn))
    k = int(rng.integers(1, max_k))
    elements = np.unique(rng.integers(-5, 6, size=k))
    weights = rng.random(len(elements)) + 0.1
    w = rng.choice(elements, size=(m, n), p=weights / weights.sum()).astype(np.float64)
    x = rng.integers(-4, 5, size=n).astype(np.float64)
    return w, x


def criterion3(seed: int):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(1, 501))
    n = int(rng.integers(1, 501))
    k = int(rng.integers(2, 129))
    elements = np.unique(rng.integers(-63, 64, size=k)).astype(np.float64)
    weights = rng.random(len(elements)) ** 3 + 1e-3
    w = rng.choice(elements, size=(m, n), p=weights / weights.sum())
    x = rng.integers(-8, 9, size=n).astype(np.float64)
    return w, x


def _quantise(values: np.ndarray, bits: int) -> np.ndarray:
    lo, hi = float(values.min()), float(values.max())
    levels = 1 << bits
    if hi == lo:
        return np.full_like(values, lo)
    step = (hi - lo) / (levels - 1)
    idx = np.clip(np.ceil((values - lo) / step - 0.5).astype(np.int64), 0, levels - 1)
    return lo + idx * step


def quantized(seed: int):
    rng = np.random.default_rng(2000 + seed)
    w = _quantise(rng.normal(size=(40, 60)), int(rng.integers(2, 8)))
    x = rng.normal(size=60)
    return w, x


def nonzero_mode(seed: int):
    rng = np.random.default_rng(3000 + seed)
    w = _quantise(rng.uniform(0.25, 2.0, size=(20, 30)), int(rng.integers(2, 8)))
    x = rng.normal(size=30)
    return w, x


def matrix_rhs(seed: int, w: np.ndarray, cols: int = 4) -> np.ndarray:
    rng = np.random.default_rng(4000 + seed)
    return rng.integers(-3, 4, size=(w.shape[1], cols)).astype(np.float64)


RECIPES = {
    "low_entropy": low_entropy,
    "criterion3": criterion3,
    "quantized": quantized,
    "nonzero_mode": nonzero_mode,
}
