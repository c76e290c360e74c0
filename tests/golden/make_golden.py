"""Generate the golden fixtures by running the REFERENCE (`lemt`) here.

Run once in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed; the GPU box never reads /root/reference):
* ``small_cases.json``   — full CER/CSER arrays + f64 dot outputs for the
  paper's 5x12 matrix M, every edge case the reference tests pin
  (tests/test_formats.py:53-139), and 40 low-entropy recipe matrices.
* ``recipe_digests.json`` — sha256 digests of every encoded array, widths,
  sizes and the f64 dot output for the larger recipe families
  (criterion-3 integer alphabets, quantised real alphabets, non-zero mode).
* ``configs.json`` + ``configs_y.npz`` — digests/sizes of the CER/CSER
  encodings of synthetic configs 1-4 and the reference
  float64 dot outputs for seeded inputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

import lemt  # noqa: E402  (the reference, from PYTHONPATH)
from lemt import DenseMatrix  # noqa: E402

import recipes  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402


def digest(arr: np.ndarray) -> str:
    arr = np.ascontiguousarray(arr)
    h = hashlib.sha256(arr.dtype.str.encode())
    h.update(arr.tobytes())
    return h.hexdigest()


def enc_full(enc) -> dict:
    out = {
        "omega": [float(v) for v in enc.omega],
        "omega_signbit": [bool(b) for b in np.signbit(enc.omega)],
        "colI": enc.col_index.tolist(),
        "omegaPtr": enc.omega_ptr.tolist(),
        "rowPtr": enc.row_ptr.tolist(),
        "bits": {"colI": enc.col_index_bits, "omegaPtr": enc.omega_ptr_bits, "rowPtr": enc.row_ptr_bits},
        "storage_bits": int(lemt.storage_bits(enc)),
    }
    if isinstance(enc, lemt.CserMatrix):
        out["omegaI"] = enc.omega_index.tolist()
        out["bits"]["omegaI"] = enc.omega_index_bits
        out["mode_index"] = int(enc.mode_index)
    return out


def enc_digest(enc) -> dict:
    out = {
        "K": len(enc.omega),
        "nnz": int(enc.nnz),
        "segments": int(enc.segment_count),
        "omega": digest(enc.omega),
        "colI": digest(enc.col_index),
        "omegaPtr": digest(enc.omega_ptr),
        "rowPtr": digest(enc.row_ptr),
        "bits": {"colI": enc.col_index_bits, "omegaPtr": enc.omega_ptr_bits, "rowPtr": enc.row_ptr_bits},
        "storage_bits": int(lemt.storage_bits(enc)),
    }
    if isinstance(enc, lemt.CserMatrix):
        out["omegaI"] = digest(enc.omega_index)
        out["bits"]["omegaI"] = enc.omega_index_bits
        out["mode_index"] = int(enc.mode_index)
    return out


def run_case(name, w, x, background=None, index_bits="auto", full=True):
    a = DenseMatrix(w)
    case = {"name": name, "background": background, "index_bits": index_bits}
    if full:
        case["matrix"] = [[float(v) for v in row] for row in np.asarray(w)]
        case["x"] = np.asarray(x).tolist()
    for kind, encode in (("cer", lemt.encode_cer), ("cser", lemt.encode_cser)):
        try:
            enc = encode(a, index_bits=index_bits, background=background)
        except Exception as ex:  # the reference's error behaviour is part of the contract
            case[kind] = {"error": type(ex).__name__, "message": str(ex)}
            continue
        case[kind] = enc_full(enc) if full else enc_digest(enc)
        y = lemt.dot(enc, np.asarray(x, dtype=np.float64))
        if full:
            case[kind]["y"] = np.asarray(y).tolist()
        else:
            case[kind]["y_digest"] = digest(np.asarray(y))
            case[kind]["y_absmax"] = float(np.abs(y).max()) if y.size else 0.0
    case["y_dense"] = np.asarray(np.asarray(w) @ np.asarray(x, dtype=np.float64)).tolist() if full else None
    return case


REF_ROWS = [  # the paper's worked example M (tests/conftest.py:8-14)
    [0, 3, 0, 2, 4, 0, 0, 2, 3, 4, 0, 4],
    [4, 4, 0, 0, 0, 4, 0, 0, 4, 4, 0, 4],
    [4, 0, 3, 4, 0, 0, 0, 4, 0, 2, 0, 0],
    [0, 0, 0, 4, 4, 4, 0, 3, 4, 4, 0, 0],
    [0, 4, 4, 0, 0, 4, 0, 4, 0, 0, 0, 0],
]


def small_cases() -> list:
    m = np.array(REF_ROWS, dtype=float)
    cases = [
        run_case("M_ones", m, np.ones(12)),
        run_case("M_linspace", m, np.linspace(-1, 1, 12)),
        run_case("M_matrix_rhs", m, np.random.default_rng(0).integers(-3, 4, size=(12, 4)).astype(float)),
        run_case("M_bits32", m, np.ones(12), index_bits=32),
        run_case("M_bits16", m, np.ones(12), index_bits=16),
        run_case("M_bits8", m, np.ones(12), index_bits=8),
        run_case("M_bg3", m, np.arange(12.0), background=3.0),
        run_case("M_bg_absent", m, np.arange(12.0), background=7.5),
        run_case("zero_3x3", np.zeros((3, 3)), np.arange(3.0)),
        run_case("zero_2x2", np.zeros((2, 2)), np.arange(2.0)),
        run_case("one_by_one", np.array([[5.0]]), np.array([2.0])),
        run_case("padding_rule", np.array([[0, 1, 1], [0, 2, 0], [1, 2, 0]], float), np.array([1.0, 2.0, 3.0])),
        run_case("constant_row_default_bg", np.array([[4, 4, 4]], float), np.array([1.0, 2.0, 3.0])),
        run_case("constant_row_bg0", np.array([[4, 4, 4]], float), np.array([1.0, 2.0, 3.0]), background=0.0),
        run_case("cser_nonzero_mode", np.array([[5, 5, 1], [5, 1, 5]], float), np.array([1.0, -1.0, 2.0])),
        run_case("identity", np.eye(3), np.array([1.0, 2.0, 3.0])),
        run_case("empty_rows", np.array([[1, 1], [0, 0], [0, 0], [2, 1]], float), np.array([1.0, 2.0])),
        run_case("neg_zero_only", np.array([[-0.0, -0.0, 1.0]]), np.array([1.0, 2.0, 3.0])),
        run_case("neg_zero_bg", np.array([[0.0, 2.0, 2.0]]), np.array([1.0, 2.0, 3.0]), background=-0.0),
        run_case("explicit_bg_mid", np.array([[3, 2, 2, 1]], float), np.array([1.0, 2.0, 3.0, 4.0]), background=2.0),
        run_case("bits8_overflow", np.zeros((2, 300)) + np.eye(2, 300), np.ones(300), index_bits=8),
        run_case("bad_bits", m, np.ones(12), index_bits=12),
        run_case("wide_row_300", (np.arange(600).reshape(2, 300) % 7 == 0).astype(float) * 3.0, np.ones(300)),
        run_case("inf_values", np.array([[np.inf, 1, 1, -np.inf], [1, 1, 0, np.inf]]), np.array([0.0, 1.0, 1.0, 0.0])),
    ]
    for seed in range(40):
        w, x = recipes.low_entropy(seed)
        cases.append(run_case(f"low_entropy_{seed}", w, x))
    for seed in range(3):
        w, _ = recipes.low_entropy(100 + seed, max_mn=12)
        cases.append(run_case(f"low_entropy_rhs_{seed}", w, recipes.matrix_rhs(seed, w)))
    return cases


def recipe_digests() -> dict:
    out = {}
    families = {"criterion3": 30, "quantized": 20, "nonzero_mode": 20}
    for fam, count in families.items():
        out[fam] = []
        for seed in range(count):
            w, x = recipes.RECIPES[fam](seed)
            case = run_case(f"{fam}_{seed}", w, x, full=False)
            case["seed"] = seed
            case["shape"] = list(w.shape)
            out[fam].append(case)
    return out


def config_goldens():
    meta, ys = {}, {}
    for name in ("oracle", "alexnet-fc6", "vgg-fc6", "resnet-conv"):
        t0 = time.time()
        cfg = synth.config(name)
        w, _ = synth.make_layer(cfg)
        a = DenseMatrix(w)
        entry = {"m": cfg.m, "n": cfg.n}
        # seeded B=1 probe input, independent of the config's own X draws
        x1 = np.random.default_rng(1).standard_normal(cfg.n, dtype=np.float32)
        for kind, encode in (("cer", lemt.encode_cer), ("cser", lemt.encode_cser)):
            enc = encode(a)
            entry[kind] = enc_digest(enc)
            y = lemt.dot(enc, x1.astype(np.float64))
            ys[f"{name}/{kind}/b1"] = y
            if name == "oracle":
                xb = np.random.default_rng(2).standard_normal((cfg.n, 8), dtype=np.float32)
                ys[f"{name}/{kind}/b8"] = lemt.dot(enc, xb.astype(np.float64))
        meta[name] = entry
        print(f"  {name}: {time.time() - t0:.1f}s", flush=True)
    return meta, ys


def main():
    print("small cases ...", flush=True)
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "lemt " + lemt.__version__,
                   "numpy": np.__version__, "cases": small_cases()}, f)
    print("recipe digests ...", flush=True)
    with open(os.path.join(HERE, "recipe_digests.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "lemt " + lemt.__version__,
                   "numpy": np.__version__, "families": recipe_digests()}, f, indent=0)
    print("configs ...", flush=True)
    meta, ys = config_goldens()
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "lemt " + lemt.__version__,
                   "numpy": np.__version__, "seed": 0, "probe_x": "default_rng(1).standard_normal(n, float32); "
                   "oracle b8: default_rng(2).standard_normal((n,8), float32)", "configs": meta}, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "configs_y.npz"), **ys)


if __name__ == "__main__":
    main()
