"""One dot call (mat-vec or mat-mat, for ncu): python tools/mm_one.py config batch kind [calls]; the kernel variant comes from
MM_PATH (auto / flat / segment / tiled) and MV_PATH (auto / window / tile / run), pinned with cerdot_set_kernel_path.
The first call warms up (and builds the mat-mat's tile view); profile with --launch-skip accordingly."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200 import synth  # noqa: E402
from paper_1805_10692_b200._native import force_path  # noqa: E402


def main():
    name, batch, kind = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    calls = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    cfg = synth.config(name)
    rng = np.random.default_rng(0)
    if cfg.m * cfg.n > 10**9:
        w = synth.make_weights_device(cfg, 0, "cuda")
    else:
        w = torch.from_numpy(synth.make_weights(cfg, rng)).cuda()
    x = torch.from_numpy(synth.make_inputs(cfg, rng, batch)).cuda()
    enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
    del w
    y = torch.empty((cfg.m, batch) if batch > 1 else (cfg.m,), device="cuda")
    with force_path("matmat", os.environ.get("MM_PATH", "auto")), force_path("matvec", os.environ.get("MV_PATH", "auto")), \
            force_path("matmat_split", int(os.environ.get("MM_SPLIT", "0"))), \
            force_path("matmat_tile", int(os.environ.get("MM_TILE", "0"))):
        for _ in range(calls):
            cd.dot_device(enc, x, out=y)
    torch.cuda.synchronize()
    print("ok", float(y.abs().sum()))


if __name__ == "__main__":
    main()
