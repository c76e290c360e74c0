"""Conversion time per config (device-synchronised wall time of encode_cer / encode_cser, best of N)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402


def main():
    for name in sys.argv[1:] or ["alexnet-fc6", "vgg-fc6", "resnet-conv"]:
        cfg = synth.config(name)
        w = (synth.make_weights_device(cfg, 0, "cuda") if cfg.m * cfg.n > 10**9
             else torch.from_numpy(synth.make_weights(cfg, np.random.default_rng(0))).cuda())
        for kind, enc in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
            enc(w)
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(5):
                t0 = time.perf_counter()
                enc(w)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(json.dumps({"config": name, "kind": kind, "ms": round(best * 1e3, 3),
                              "dense_gbs": round(w.numel() * 4 / best / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
