"""Measured parity of every timed configuration / input / kernel path against the float64 C oracle
(max|y - y_ref| / max|y_ref|, the reference tests' metric), as one JSON object for DESIGN.md §4.

    python tools/parity_table.py > profiles/r02_parity_table.json      (GPU box)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from oracle import c_oracle, numpy_port  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402
from paper_1805_10692_b200._native import force_path  # noqa: E402


def err(y, ref):
    y = np.asarray(y, dtype=np.float64)
    return float(np.abs(y - ref).max() / np.abs(ref).max())


def main():
    out = {"metric": "max|y - y_ref| / max|y_ref| vs the float64 C oracle (cer_oracle.c)", "b1": {}, "batch": {}}
    for name in ("oracle", "alexnet-fc6", "vgg-fc6", "resnet-conv"):
        cfg = synth.config(name)
        w, xs = synth.make_layer(cfg)
        wt = torch.from_numpy(w).cuda()
        rng = np.random.default_rng(77)
        inputs = {"own": synth.make_inputs(cfg, synth.rng_after_weights(cfg, 0), 1),
                  "normal": rng.standard_normal(cfg.n, dtype=np.float32),
                  "abs_normal": np.abs(rng.standard_normal(cfg.n, dtype=np.float32)),
                  "ones": np.ones(cfg.n, dtype=np.float32)}
        for kind in ("cer", "cser"):
            enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
            ref_enc = c_oracle.encode(w, kind)
            for tag, x in inputs.items():
                ref = c_oracle.dot(ref_enc, x.astype(np.float64))
                for path in ("window", "tile", "run", "stream", "row"):
                    with force_path("matvec", path):
                        y = cd.dot(enc, torch.from_numpy(x).cuda()).cpu().numpy()
                    out["b1"][f"{name}/{kind}/{tag}/{path}"] = err(y, ref)
            for b in cfg.batches:
                if b == 1:
                    continue
                x = xs[b]
                ref = c_oracle.dot(ref_enc, x.astype(np.float64))
                for path in ("flat", "tiled", "tiled_frag"):
                    with force_path("matmat", path):
                        y = cd.dot(enc, torch.from_numpy(x).cuda()).cpu().numpy()
                    out["batch"][f"{name}/{kind}/B={b}/{path}"] = err(y, ref)
        del wt
        torch.cuda.empty_cache()
    # config 5: B=1 every row, B=256 on eight spread 64-row blocks
    cfg = synth.config("large")
    w = synth.make_weights_device(cfg, 0, "cuda")
    encs = {"cer": cd.encode_cer(w), "cser": cd.encode_cser(w)}
    wh = w.cpu().numpy()
    del w
    torch.cuda.empty_cache()
    x = synth.make_inputs(cfg, synth.rng_after_weights(cfg, 0), 256)
    x1 = np.ascontiguousarray(x[:, 0])
    for kind, enc in encs.items():
        ref_enc = c_oracle.encode(wh, kind)
        ref1 = c_oracle.dot(ref_enc, x1.astype(np.float64))
        for path in ("window", "run", "stream"):
            with force_path("matvec", path):
                y = cd.dot(enc, torch.from_numpy(x1).cuda()).cpu().numpy()
            out["b1"][f"large/{kind}/own/{path}"] = err(y, ref1)
        for path in ("flat", "tiled", "tiled_frag"):
            with force_path("matmat", path):
                y = cd.dot(enc, torch.from_numpy(x).cuda()).cpu().numpy()
            worst = 0.0
            for r0 in (0, 4100, 8200, 12300, 16400, 20500, 24600, cfg.m - 64):
                blk = numpy_port.row_block(ref_enc, r0, r0 + 64)
                worst = max(worst, err(y[r0:r0 + 64], c_oracle.dot(blk, x.astype(np.float64))))
            out["batch"][f"large/{kind}/B=256 (8 x 64 rows)/{path}"] = worst
    out["worst_b1"] = max(out["b1"].values())
    out["worst_batch"] = max(out["batch"].values())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
