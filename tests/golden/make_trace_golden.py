"""Generate the analytic-trace and cost-model fixtures by running the REFERENCE (`lemt`) here.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_trace_golden.py

Output (committed; the GPU box never reads /root/reference): ``traces.json`` -- for the CER and CSER
encodings of synthetic configs 1-4, at B=1 and at each config's BASELINE batch
(``columns``), and for two non-zero-background cases:
* the reference's full OpTrace counts (lemt.kernels.trace_of, kernels.py:175-234), and
* lemt.costmodel.price_trace of that trace (costmodel.py:179-217) under the default energy table with
  per-array tiers from lemt.formats.array_bytes, and under the unit table at a fixed tier -- the
  numbers the drop-in's OpTrace must reproduce when fed to price_trace (bench_matrix's path).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import lemt  # noqa: E402  (the reference, from PYTHONPATH)
from lemt import DenseMatrix, costmodel, formats, kernels  # noqa: E402

from paper_1805_10692_b200 import synth  # noqa: E402


def counts_list(trace) -> list:
    return sorted([k[0], int(k[1]), k[2], int(v)] for k, v in trace.counts.items())


def prices(trace, enc) -> dict:
    sizes = formats.array_bytes(enc)
    rep = costmodel.price_trace(trace, costmodel.default_energy_table(), array_sizes=dict(sizes))
    unit = costmodel.price_trace(trace, costmodel.unit_table(), fixed_tier="<32KB")
    return {"default_energy_total": rep.total, "default_energy_unit": rep.unit,
            "default_energy_breakdown": sorted([k[0], k[1], v] for k, v in rep.breakdown.items()),
            "array_sizes": {k: float(v) for k, v in sizes.items()},
            "unit_32KB_total": unit.total}


def main():
    out = {"_generator": "tests/golden/make_trace_golden.py (lemt " + getattr(lemt, "__version__", "?") + ")",
           "cases": {}}
    for name in ("oracle", "alexnet-fc6", "vgg-fc6", "resnet-conv"):
        cfg = synth.config(name)
        w, _ = synth.make_layer(cfg)
        dm = DenseMatrix(w.astype(np.float64))
        for kind, enc_fn in (("cer", lemt.encode_cer), ("cser", lemt.encode_cser)):
            enc = enc_fn(dm)
            for cols in sorted({1, *cfg.batches}):
                t = kernels.trace_of(enc, columns=cols)
                out["cases"][f"{name}/{kind}/{cols}"] = {"config": name, "kind": kind, "columns": cols,
                                                         "counts": counts_list(t), **prices(t, enc)}
            print(name, kind, flush=True)
    # non-zero background: an explicit background absent from the matrix, and config 4's nonzero mode
    rng = np.random.default_rng(5)
    w = rng.choice([-2.0, -1.0, 0.0, 1.0, 3.0], size=(40, 70), p=[0.1, 0.2, 0.4, 0.2, 0.1])
    for kind, enc_fn in (("cer", lemt.encode_cer), ("cser", lemt.encode_cser)):
        enc = enc_fn(DenseMatrix(w), background=0.5)
        t = kernels.trace_of(enc, columns=3)
        out["cases"][f"bg_absent/{kind}/3"] = {"matrix_seed": 5, "background": 0.5, "kind": kind, "columns": 3,
                                               "counts": counts_list(t), **prices(t, enc)}
    with open(os.path.join(HERE, "traces.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
