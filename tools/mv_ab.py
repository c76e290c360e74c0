"""A/B of mat-vec kernel variants on one config: python tools/mv_ab.py config "path[:nt]" ...  (e.g. large run stream stream:1024)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402
from paper_1805_10692_b200._native import force_path  # noqa: E402
from tools.mv_time import graph_us  # noqa: E402


def main():
    name, variants = sys.argv[1], sys.argv[2:]
    cfg = synth.config(name)
    rng = np.random.default_rng(0)
    w = synth.make_weights_device(cfg, 0, "cuda") if cfg.m * cfg.n > 10**9 else torch.from_numpy(synth.make_weights(cfg, rng)).cuda()
    x = synth.make_inputs(cfg, rng, 1)
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
        R = 16 if cfg.m * cfg.n < 10**8 else 2
        copies = [bench._clone(cd, enc) for _ in range(R)]
        xs = [torch.from_numpy(x).cuda().reshape(-1) for _ in range(R)]
        ref = None
        for var in variants:
            path, _, nt = var.partition(":")
            ys = [torch.full((cfg.m,), float("nan"), device="cuda") for _ in range(R)]
            with force_path("matvec", path), force_path("matvec_nt", int(nt or 0)):
                us = graph_us(copies, xs, ys)
            y = ys[0].double().cpu().numpy()
            ref = y if ref is None else ref
            gb = cd.storage_bits(enc) / 8 + 4 * (cfg.n + cfg.m)
            print(json.dumps({"config": name, "kind": kind, "variant": var, "us": round(us, 3), "gbs": round(gb / us / 1e3, 1),
                              "rel_vs_first": float(np.abs(y - ref).max() / np.abs(ref).max())}), flush=True)
        del copies, xs


if __name__ == "__main__":
    main()
