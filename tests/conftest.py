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


def validate_case_arrays(bases, case) -> dict:
    """The (possibly corrupted) encoding of one tests/golden/validate_cases.json case, as an oracle dict."""
    base = bases[case["base"]]
    enc = {k: (list(v) if isinstance(v, list) else v) for k, v in base.items() if k != "widths"}
    if "set" in case:
        name, pos, value = case["set"]
        enc[name][pos] = value
    if "drop" in case:
        enc[case["drop"]] = enc[case["drop"]][:-1]
    if case.get("omega_swap") and len(enc["omega"]) > 2:
        enc["omega"][1], enc["omega"][2] = enc["omega"][2], enc["omega"][1]
    if case.get("omega_dup") and len(enc["omega"]) > 1:
        enc["omega"][-1] = enc["omega"][0]
    if "mode" in case:
        enc["mode_index"] = case["mode"]
    out = {"kind": enc["kind"], "m": enc["m"], "n": enc["n"], "omega": np.asarray(enc["omega"], dtype=np.float64)}
    for k in ("colI", "omegaPtr", "rowPtr", "omegaI"):
        if k in enc:
            out[k] = np.asarray(enc[k], dtype=np.dtype(f"uint{base['widths'][k]}"))
    if "mode_index" in enc:
        out["mode_index"] = enc["mode_index"]
    return out


@pytest.fixture(scope="session")
def validate_cases():
    with open(os.path.join(GOLDEN, "validate_cases.json")) as f:
        return json.load(f)


@pytest.fixture
def kernel_path():
    """pin(op, path): force a kernel choice (cerdot_set_kernel_path) for the rest of the test."""
    from paper_1805_10692_b200 import _native

    pinned = []

    def pin(op, path):
        ctx = _native.force_path(op, path)
        ctx.__enter__()
        pinned.append(ctx)

    yield pin
    for ctx in reversed(pinned):
        ctx.__exit__(None, None, None)
