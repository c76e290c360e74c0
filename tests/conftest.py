import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(HERE, "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; run with -m gpu")


def digest(arr) -> str:
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256(arr.dtype.str.encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def small_cases():
    return _load("small_cases.json")["cases"]


@pytest.fixture(scope="session")
def recipe_digests():
    return _load("recipe_digests.json")["families"]


@pytest.fixture(scope="session")
def config_goldens():
    meta = _load("configs.json")
    ys = dict(np.load(os.path.join(GOLDEN, "configs_y.npz")))
    return meta, ys


def is_integer_case(case) -> bool:
    w = np.asarray(case["matrix"], dtype=float)
    x = np.asarray(case["x"], dtype=float)
    return bool(np.all(np.isfinite(w)) and np.all(w == np.round(w)) and np.all(x == np.round(x)))


def rel_err(y, y_ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    if y_ref.size == 0:
        return 0.0
    # the reference's own metric (tests/test_kernels.py:143-146, test_acceptance.py:136-138)
    return float(np.abs(y - y_ref).max() / (np.abs(y_ref).max() + 1e-30))


REL_TOL = 1e-5  # north_star: fp32 dot within max relative error 1e-5 of the float64 oracle


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
