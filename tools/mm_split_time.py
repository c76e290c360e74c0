"""Tiled mat-mat with the X tiles split over S CTAs per row block vs the flat kernel (graph-replayed, rotating copies).
Usage: python tools/mm_split_time.py [config:batch ...]"""
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

cases = [c.split(":") for c in (sys.argv[1:] or ["alexnet-fc6:64", "vgg-fc6:128", "resnet-conv:1568"])]
for name, b in cases:
    b = int(b)
    cfg = synth.config(name)
    if name == "large":
        wt = synth.make_weights_device(cfg, 0, torch.device("cuda"))
    else:
        wt = torch.from_numpy(synth.make_layer(cfg)[0]).cuda()
    x = synth.make_inputs(cfg, np.random.default_rng(1), b)
    enc = cd.encode_cer(wt)
    rot = 2 if name == "large" else 4
    copies = [bench._clone(cd, enc) for _ in range(rot)]
    xs = [torch.from_numpy(x).cuda() for _ in range(rot)]
    ys = [torch.empty((cfg.m, b), device="cuda") for _ in range(rot)]
    ref = None
    for path, split, nt in [("flat", 0, 0)] + [("tiled", s, t) for t in [int(v) for v in os.environ.get("MM_TILES", "128 256").split()] for s in (1, 2, 4, 8)]:
        with force_path("matmat", path), force_path("matmat_split", split), force_path("matmat_tile", nt):
            for i in range(rot):
                cd.dot_device(copies[i], xs[i], out=ys[i])
            torch.cuda.synchronize()
            steps = 3 if name == "large" else 20
            secs = bench._graph_time(lambda i: cd.dot_device(copies[i], xs[i], out=ys[i]), steps, 3, rot, torch)
        y = ys[0].double().cpu().numpy()
        ref = y if ref is None else ref
        print(json.dumps({"config": name, "batch": b, "path": path, "split": split, "nt": nt, "us": round(secs / steps * 1e6, 2),
                          "rel_vs_flat": float(np.abs(y - ref).max() / np.abs(ref).max())}), flush=True)
    del copies, xs, ys, enc, wt
    torch.cuda.empty_cache()
