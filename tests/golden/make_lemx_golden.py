"""Golden LEMX containers written by the REFERENCE (`lemt.io.write_matrix`, io.py:177-211).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_lemx_golden.py

Output (committed): ``lemx_files.json`` -- for the 5x12 matrix M and two seeded low-entropy matrices,
CER and CSER at element widths 8/16/32/64: the container bytes (hex) and the arrays they hold.  Plus
the reference's read errors for truncated / bad-magic / bad-version / trailing-byte files.
"""

from __future__ import annotations

import json
import os
import tempfile

import numpy as np

from lemt import DenseMatrix
from lemt.formats import encode_cer, encode_cser
from lemt.io import IoFormatError, read_matrix, write_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
M = [[0, 3, 0, 2, 4, 0, 0, 2, 3, 4, 0, 4], [4, 4, 0, 0, 0, 4, 0, 0, 4, 4, 0, 4], [4, 0, 3, 4, 0, 0, 0, 4, 0, 2, 0, 0],
     [0, 0, 0, 4, 4, 4, 0, 3, 4, 4, 0, 0], [0, 4, 4, 0, 0, 4, 0, 4, 0, 0, 0, 0]]


def main():
    mats = [np.array(M, dtype=float)]
    for seed in (5, 9):
        r = np.random.default_rng(seed)
        m, n = int(r.integers(6, 14)), int(r.integers(20, 90))
        elems = np.unique(r.integers(-5, 6, size=6)).astype(float)
        w = r.random(len(elems)) + 0.1
        mats.append(r.choice(elems, size=(m, n), p=w / w.sum()))
    files, errors = [], []
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.lemx")
        for mi, w in enumerate(mats):
            for bits in (8, 16, 32, 64):
                for kind, encode in (("cer", encode_cer), ("cser", encode_cser)):
                    enc = encode(DenseMatrix(w, element_bits=bits))
                    write_matrix(path, enc)
                    raw = open(path, "rb").read()
                    rec = {"matrix": mi, "element_bits": bits, "kind": kind, "hex": raw.hex(),
                           "m": enc.m, "n": enc.n, "omega": enc.omega.tolist(), "colI": enc.col_index.tolist(),
                           "omegaPtr": enc.omega_ptr.tolist(), "rowPtr": enc.row_ptr.tolist(),
                           "widths": [enc.col_index_bits, enc.omega_ptr_bits, enc.row_ptr_bits]}
                    if kind == "cser":
                        rec["omegaI"] = enc.omega_index.tolist()
                        rec["mode_index"] = enc.mode_index
                        rec["widths"].append(enc.omega_index_bits)
                    files.append(rec)
        base = bytes.fromhex(files[2]["hex"])  # M, 16-bit elements, CER
        for label, blob in (("truncated", base[:-3]), ("bad-magic", b"XEMX" + base[4:]),
                            ("bad-version", base[:4] + b"\x07\x00" + base[6:]), ("trailing", base + b"\x00"),
                            ("short-header", base[:9])):
            open(path, "wb").write(blob)
            try:
                read_matrix(path)
                errors.append({"label": label, "hex": blob.hex(), "code": None})
            except IoFormatError as err:
                errors.append({"label": label, "hex": blob.hex(), "code": err.code})
            except Exception as err:  # struct.error on a header shorter than the fixed fields
                errors.append({"label": label, "hex": blob.hex(), "code": type(err).__name__})
    with open(os.path.join(HERE, "lemx_files.json"), "w") as f:
        json.dump({"files": files, "errors": errors}, f, separators=(",", ":"))
    print(len(files), "files;", [(e["label"], e["code"]) for e in errors])


if __name__ == "__main__":
    main()
