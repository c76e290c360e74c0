"""Randomised stress of every dot kernel path on integer data (bitwise vs numpy w @ x): random shapes, densities,
alphabet sizes, backgrounds; B = 1 through the window / tile / run / stream / row kernels, B > 1 through the flat
and tiled kernels (tile rows 128 / 256 x 1 / 2 / 4 CTAs per row block).  Usage: python tools/stress_paths.py [trials] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1805_10692_b200 as cd  # noqa: E402
from paper_1805_10692_b200._native import force_path  # noqa: E402


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    checks = 0
    for t in range(trials):
        m = int(rng.integers(1, 260))
        n = int(rng.choice([16, 48, 255, 256, 1000, 2048, 4100, 9000]))
        levels = int(rng.choice([2, 3, 9, 40, 300, 600]))
        p0 = float(rng.choice([0.3, 0.7, 0.92, 0.99]))
        vals = np.arange(-(levels // 2), levels - levels // 2).astype(np.float64)
        p = rng.random(levels) + 0.02
        p = p / p.sum() * (1 - p0)
        p[levels // 2] += p0
        w = rng.choice(vals, size=(m, n), p=p / p.sum())
        if m > 3:
            w[int(rng.integers(0, m))] = 0.0
            w[int(rng.integers(0, m))] = vals[-1]
        bg = None if rng.random() < 0.6 else float(rng.choice(vals))
        batch = int(rng.choice([2, 40, 64, 100]))
        x1 = rng.integers(-2, 3, size=n).astype(np.float64)
        xb = rng.integers(-2, 3, size=(n, batch)).astype(np.float64)
        xbt = torch.from_numpy(xb.astype(np.float32)).cuda()
        for encode in (cd.encode_cer, cd.encode_cser):
            enc = encode(w, background=bg)
            tag = (t, m, n, levels, p0, bg, encode.__name__)
            for path in ("window", "tile", "run", "stream", "row"):
                with force_path("matvec", path):
                    assert np.array_equal(cd.dot(enc, x1), w @ x1), tag + (path,)
                    checks += 1
            want = w @ xb
            with force_path("matmat", "flat"):
                assert np.array_equal(cd.dot(enc, xbt).cpu().numpy(), want), tag + ("flat", batch)
            for nt in (128, 256):
                for split in (1, 2, 4):
                    with force_path("matmat", "tiled"), force_path("matmat_tile", nt), force_path("matmat_split", split):
                        assert np.array_equal(cd.dot(enc, xbt).cpu().numpy(), want), tag + ("tiled", nt, split, batch)
                        checks += 1
            assert np.array_equal(cd.dot(enc, xbt).cpu().numpy(), want), tag + ("auto", batch)
    print("stress ok:", trials, "matrices,", checks, "kernel checks")


if __name__ == "__main__":
    main()
