"""Graph-replayed cold mat-vec time (us per call) for each config x kind; prints one JSON line per case.

Usage: python tools/mv_time.py [config ...]   (CERDOT_LIB selects the library for A/B runs)
MV_VARIANTS="1 3" times each mat-vec kernel path (cerdot_set_kernel_path: 1 window, 2 tile, 3 run; "auto")
in one process and reports each variant's max|y - y_first| / max|y_first| against the first.
"""
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


def graph_us(encs, xs, ys, reps=20):
    R = len(encs)
    g = torch.cuda.CUDAGraph()
    for i in range(R):
        cd.dot_device(encs[i], xs[i], out=ys[i])
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(R):
            cd.dot_device(encs[i], xs[i], out=ys[i])
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / (reps * R)


def main():
    names = sys.argv[1:] or ["alexnet-fc6", "vgg-fc6", "resnet-conv"]
    tag = os.environ.get("CERDOT_LIB", "tree")
    for name in names:
        cfg = synth.config(name)
        rng = np.random.default_rng(0)
        if cfg.m * cfg.n > 10**9:
            w = synth.make_weights_device(cfg, 0, "cuda")
        else:
            w = torch.from_numpy(synth.make_weights(cfg, rng)).cuda()
        x = synth.make_inputs(cfg, rng, 1)
        for kind in ("cer", "cser"):
            enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
            R = 16 if cfg.m * cfg.n < 10**8 else 2
            copies = [bench._clone(cd, enc) for _ in range(R)]
            xs = [torch.from_numpy(x).cuda().reshape(-1) for _ in range(R)]
            ref = None
            for var in os.environ.get("MV_VARIANTS", "auto").split():
                ys = [torch.full((cfg.m,), float("nan"), device="cuda") for _ in range(R)]
                with force_path("matvec", 0 if var == "auto" else int(var)):
                    us = graph_us(copies, xs, ys)
                y = ys[0].double().cpu().numpy()
                if ref is None:
                    ref = y
                err = float(np.abs(y - ref).max() / np.abs(ref).max())
                gb = cd.storage_bits(enc) / 8 + 4 * (cfg.n + cfg.m)
                print(json.dumps({"lib": os.path.basename(tag), "config": name, "kind": kind, "variant": var,
                                  "us": round(us, 3), "gbs": round(gb / us / 1e3, 1), "rel_vs_first": err}),
                      flush=True)
            del copies, xs


if __name__ == "__main__":
    main()
