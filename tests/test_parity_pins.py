"""GPU parity pins on every configuration and input the benchmark times (VERDICT r1 "next" #1).

* Config 5 (32768^2, K=256), the seeded numpy matrix drawn on the device (bit-identical, see
  test_gpu_parity.test_device_draw_equals_numpy_draw):
  - conversion: omega, colI, omegaPtr, rowPtr, omegaI, mode_index and the auto widths of the GPU
    encodings equal the C oracle's (cer_oracle.c, pinned bit-exact to lemt on configs 1-4) on the whole
    matrix (formats.py:227-295);
  - B=256 (the bench's X, drawn after W): eight 64-row blocks spread over the matrix against the oracle
    (rows are independent; a row block of the oracle encoding is a slice, shard.slice_rows' rule);
  - B=1: every row, through the window and long-row mat-vec kernels.
* ReLU inputs at B=1 (the bench times VGG fc6 and ResNet conv B=1 with the configs' own ReLU x) and
  adversarial all-positive inputs (|N(0,1)|, all ones), through every mat-vec kernel.
* Configs 2 and 3 at their BASELINE batches through the automatic mat-mat path, every column.
Bar: max|y - y_ref| / max|y_ref| <= 1e-5 (kernels.py tests' own metric), y_ref the float64 oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import REL_TOL, has_gpu, rel_err

pytestmark = pytest.mark.gpu

if has_gpu():
    import torch

    import paper_1805_10692_b200 as cd
    from oracle import c_oracle, numpy_port
    from paper_1805_10692_b200 import synth
    from paper_1805_10692_b200._native import force_path


@pytest.fixture(scope="module")
def large_layer():
    """(host W, GPU encodings, oracle encodings, X256) of config 5, built once for the module."""
    cfg = synth.config("large")
    w = synth.make_weights_device(cfg, 0, "cuda")
    encs = {"cer": cd.encode_cer(w), "cser": cd.encode_cser(w)}
    w_host = w.cpu().numpy()
    del w
    torch.cuda.empty_cache()
    refs = {kind: c_oracle.encode(w_host, kind) for kind in ("cer", "cser")}
    x = synth.make_inputs(cfg, synth.rng_after_weights(cfg, 0), 256)
    yield cfg, encs, refs, x
    del encs, refs
    torch.cuda.empty_cache()


def test_large_conversion_bit_exact(large_layer):
    _, encs, refs, _ = large_layer
    for kind, enc in encs.items():
        ref = refs[kind]
        assert np.array_equal(enc.omega, ref["omega"]), kind
        for name, field in (("colI", "col_index"), ("omegaPtr", "omega_ptr"), ("rowPtr", "row_ptr"),
                            ("omegaI", "omega_index")):
            if name not in ref:
                continue
            got = getattr(enc, field)
            assert got.dtype == ref[name].dtype, (kind, name, got.dtype, ref[name].dtype)
            assert np.array_equal(got, ref[name]), (kind, name)
        if kind == "cser":
            assert enc.mode_index == ref["mode_index"]


def test_large_b256_rows_spread(large_layer):
    cfg, encs, refs, x = large_layer
    xt = torch.from_numpy(x).cuda()
    starts = [0, 4100, 8200, 12300, 16400, 20500, 24600, cfg.m - 64]
    for kind, enc in encs.items():
        y = cd.dot(enc, xt).cpu().numpy()
        for r0 in starts:
            blk = numpy_port.row_block(refs[kind], r0, r0 + 64)
            ref = c_oracle.dot(blk, x.astype(np.float64))
            err = rel_err(y[r0:r0 + 64], ref)
            assert err <= REL_TOL, (kind, r0, err)


@pytest.mark.parametrize("path", ["window", "run", "stream"])
def test_large_b1_every_row(large_layer, path):
    _, encs, refs, x = large_layer
    x1 = np.ascontiguousarray(x[:, 0])
    for kind, enc in encs.items():
        ref = c_oracle.dot(refs[kind], x1.astype(np.float64))
        with force_path("matvec", path):
            y = cd.dot(enc, torch.from_numpy(x1).cuda()).cpu().numpy()
        assert rel_err(y, ref) <= REL_TOL, (kind, path)


def _b1_inputs(cfg):
    """The config's own B=1 input (ReLU for VGG / ResNet) and two adversarial all-positive ones."""
    x_own = synth.make_inputs(cfg, synth.rng_after_weights(cfg, 0), 1)
    rng = np.random.default_rng(77)
    return {"own": x_own, "abs_normal": np.abs(rng.standard_normal(cfg.n, dtype=np.float32)),
            "ones": np.ones(cfg.n, dtype=np.float32)}


@pytest.mark.parametrize("path", ["window", "tile", "run", "stream", "row"])
@pytest.mark.parametrize("name", ["vgg-fc6", "resnet-conv", "alexnet-fc6"])
def test_b1_relu_and_positive_inputs(name, path):
    cfg = synth.config(name)
    w, _ = synth.make_layer(cfg)
    wt = torch.from_numpy(w).cuda()
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
        ref_enc = c_oracle.encode(w, kind)
        for tag, x in _b1_inputs(cfg).items():
            ref = c_oracle.dot(ref_enc, x.astype(np.float64))
            with force_path("matvec", path):
                y = cd.dot(enc, torch.from_numpy(x).cuda()).cpu().numpy()
            err = rel_err(y, ref)
            assert err <= REL_TOL, (name, kind, path, tag, err)


@pytest.mark.parametrize("name,batch", [("alexnet-fc6", 64), ("vgg-fc6", 128)])
def test_fc_matmat_full_batch_auto_path(name, batch):
    cfg = synth.config(name)
    w, xs = synth.make_layer(cfg)
    x = xs[batch]
    wt = torch.from_numpy(w).cuda()
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
        y = cd.dot(enc, torch.from_numpy(x).cuda()).cpu().numpy()
        ref = c_oracle.dot(c_oracle.encode(w, kind), x.astype(np.float64))
        assert rel_err(y, ref) <= REL_TOL, (name, kind)
