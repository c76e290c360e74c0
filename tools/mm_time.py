"""Mat-mat (B > 1) A/B: graph-replayed cold us per call for each kernel variant, plus a bitwise check of
every variant against the first one.  All mat-mat kernels compute each column in the same fp32 order, so
their outputs must be identical.

Usage: python tools/mm_time.py [config:batch ...]
Variants: MM_VARIANTS="1 2 3 ..." pins the mat-mat kernel (cerdot_set_kernel_path: 1 flat, 2 per-segment,
3 tiled, 4 tiled sum-then-multiply; "auto" = 0).
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


def set_variant(v: str):
    from paper_1805_10692_b200._native import lib

    lib().cerdot_set_kernel_path(1, 0 if v == "auto" else int(v))  # CERDOT_PATH_MATMAT


def graph_us(encs, xs, ys, reps=5):
    R = len(encs)
    for i in range(R):
        cd.dot_device(encs[i], xs[i], out=ys[i])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
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
    cases = sys.argv[1:] or ["alexnet-fc6:64", "vgg-fc6:128", "resnet-conv:1568"]
    variants = os.environ.get("MM_VARIANTS", "0 auto").split()
    for case in cases:
        name, _, b = case.partition(":")
        batch = int(b)
        cfg = synth.config(name)
        rng = np.random.default_rng(0)
        if cfg.m * cfg.n > 10**9:
            w = synth.make_weights_device(cfg, 0, "cuda")
        else:
            w = torch.from_numpy(synth.make_weights(cfg, rng)).cuda()
        x = synth.make_inputs(cfg, rng, batch)
        for kind in ("cer", "cser"):
            enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
            R = int(os.environ.get("MM_R", "4"))
            copies = [bench._clone(cd, enc) for _ in range(R)]
            xs = [torch.from_numpy(x).cuda() for _ in range(R)]
            ref = None
            for v in variants:
                set_variant(v)
                ys = [torch.full((cfg.m, batch), float("nan"), device="cuda") for _ in range(R)]
                us = graph_us(copies, xs, ys)
                y = ys[0].cpu().numpy()
                if ref is None:
                    ref = y
                same = bool(np.array_equal(y.view(np.uint32), ref.view(np.uint32)))
                print(json.dumps({"config": name, "batch": batch, "kind": kind, "variant": v, "us": round(us, 2),
                                  "adds_T": round(enc.nnz * batch / us / 1e6, 3), "bitwise_eq_ref": same}),
                      flush=True)
            del copies, xs
        del w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
