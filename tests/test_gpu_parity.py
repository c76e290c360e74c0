"""GPU parity: the CUDA path (through libcerdot's C ABI) against the pinned oracle.

Bars (north_star): conversion outputs bit-exact (omega, colI, omegaPtr,
rowPtr, omegaI, mode_index, auto widths); dot within max relative error
1e-5 of the float64 reference; integer alphabets bitwise (every partial sum
is an exactly representable fp32 integer, so any summation order is exact).
"""

import numpy as np
import pytest

import paper_1805_10692_b200 as cd
import recipes
from conftest import REL_TOL, digest, is_integer_case, rel_err
from oracle import c_oracle, numpy_port
from paper_1805_10692_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _assert_same(enc, g, kind, name):
    assert enc.omega.tolist() == g["omega"], name
    assert enc.col_index.tolist() == g["colI"], name
    assert enc.omega_ptr.tolist() == g["omegaPtr"], name
    assert enc.row_ptr.tolist() == g["rowPtr"], name
    assert enc.col_index_bits == g["bits"]["colI"], name
    assert enc.omega_ptr_bits == g["bits"]["omegaPtr"], name
    assert enc.row_ptr_bits == g["bits"]["rowPtr"], name
    assert cd.storage_bits(enc) == g["storage_bits"], name
    if kind == "cser":
        assert enc.omega_index.tolist() == g["omegaI"], name
        assert enc.omega_index_bits == g["bits"]["omegaI"], name
        assert enc.mode_index == g["mode_index"], name
    # the sign of a zero in omega is pinned where the reference is unambiguous
    # (single-signed zeros, or an explicit background); see DESIGN.md
    assert np.signbit(enc.omega).tolist() == g["omega_signbit"], name


def test_small_cases(small_cases):
    for case in small_cases:
        w = np.asarray(case["matrix"], dtype=float)
        x = np.asarray(case["x"], dtype=float)
        for kind in ("cer", "cser"):
            g = case[kind]
            encode = cd.encode_cer if kind == "cer" else cd.encode_cser
            if "error" in g:
                with pytest.raises(Exception) as err:
                    encode(cd.DenseMatrix(w), index_bits=case["index_bits"], background=case["background"])
                assert type(err.value).__name__ == g["error"], case["name"]
                continue
            enc = encode(cd.DenseMatrix(w), index_bits=case["index_bits"], background=case["background"])
            _assert_same(enc, g, kind, case["name"])
            y = cd.dot(enc, x)
            y_ref = np.asarray(g["y"], dtype=float)
            assert y.shape == y_ref.shape
            if not np.all(np.isfinite(y_ref)):
                assert np.array_equal(np.isnan(y), np.isnan(y_ref)), case["name"]
                continue
            if is_integer_case(case):
                assert np.array_equal(y, y_ref), (case["name"], kind, y, y_ref)
            else:
                assert rel_err(y, y_ref) <= REL_TOL, (case["name"], kind)


def test_recipe_families(recipe_digests):
    for fam, cases in recipe_digests.items():
        for case in cases:
            w, x = recipes.RECIPES[fam](case["seed"])
            for kind in ("cer", "cser"):
                g = case[kind]
                enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(w)
                tag = (fam, case["seed"], kind)
                assert digest(enc.omega) == g["omega"], tag
                assert digest(enc.col_index) == g["colI"], tag
                assert digest(enc.omega_ptr) == g["omegaPtr"], tag
                assert digest(enc.row_ptr) == g["rowPtr"], tag
                if kind == "cser":
                    assert digest(enc.omega_index) == g["omegaI"], tag
                    assert enc.mode_index == g["mode_index"], tag
                y = cd.dot(enc, x)
                if fam == "criterion3":  # integer alphabets: bitwise (tests/test_acceptance.py:108-126)
                    assert digest(y) == g["y_digest"], tag
                else:
                    ref = numpy_port.encode_cer(w) if kind == "cer" else numpy_port.encode_cser(w)
                    assert rel_err(y, numpy_port.dot(ref, x)) <= REL_TOL, tag


@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6", "vgg-fc6", "resnet-conv"])
def test_config_encodings_and_matvec(config_goldens, name):
    meta, ys = config_goldens
    w, _ = synth.make_layer(name)
    wt = torch.from_numpy(w).cuda()
    x1 = np.random.default_rng(1).standard_normal(w.shape[1], dtype=np.float32)
    outs = {}
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
        g = meta["configs"][name][kind]
        assert (enc.nnz, enc.segment_count, len(enc.omega)) == (g["nnz"], g["segments"], g["K"])
        assert digest(enc.omega) == g["omega"]
        assert digest(enc.col_index) == g["colI"]
        assert digest(enc.omega_ptr) == g["omegaPtr"]
        assert digest(enc.row_ptr) == g["rowPtr"]
        if kind == "cser":
            assert digest(enc.omega_index) == g["omegaI"]
            assert enc.mode_index == g["mode_index"]
        assert cd.storage_bits(enc) == g["storage_bits"]
        y = cd.dot(enc, x1)
        assert rel_err(y, ys[f"{name}/{kind}/b1"]) <= REL_TOL, (name, kind)
        outs[kind] = y
    # CER and CSER hold the same non-empty segments in the same order
    assert rel_err(outs["cer"], outs["cser"]) <= REL_TOL


@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6", "vgg-fc6", "resnet-conv"])
def test_config_matmat(name):
    cfg = synth.config(name)
    w, xs = synth.make_layer(cfg)
    b = max(cfg.batches)
    if b == 1:
        b = 8
        x = np.random.default_rng(2).standard_normal((cfg.n, b), dtype=np.float32)
    else:
        x = xs[b]
    if b > 256:  # keep the float64 oracle bounded: a column slice is bitwise the same computation per column
        x = np.ascontiguousarray(x[:, :200])
    wt = torch.from_numpy(w).cuda()
    xt = torch.from_numpy(x).cuda()
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
        y = cd.dot(enc, xt).cpu().numpy()
        ref = c_oracle.dot(c_oracle.encode(w, kind), x.astype(np.float64))
        assert rel_err(y, ref) <= REL_TOL, (name, kind, rel_err(y, ref))
        # column-wise parity too (each output column is its own dot product)
        col_err = np.abs(y - ref).max(axis=0) / (np.abs(ref).max(axis=0) + 1e-30)
        assert col_err.max() <= 1e-4


def test_full_batch_resnet_conv_properties():
    """Config 4 at its full B=1568: linearity and column-slice consistency (size-independent checks)."""
    cfg = synth.config("resnet-conv")
    w, xs = synth.make_layer(cfg)
    x = torch.from_numpy(xs[1568]).cuda()
    enc = cd.encode_cser(torch.from_numpy(w).cuda())
    from paper_1805_10692_b200._native import force_path

    y = cd.dot(enc, x)
    # per-column computation is independent of the batch at a fixed tile split (a narrow batch lets the
    # automatic choice split the X tiles over CTAs, which re-associates the tile partial sums)
    with force_path("matmat_split", 1):
        assert torch.equal(cd.dot(enc, x)[:, 1000:1100], cd.dot(enc, x[:, 1000:1100].contiguous()))
    y_slice = cd.dot(enc, x[:, 1000:1100].contiguous())
    assert rel_err(y_slice.cpu().numpy(), y[:, 1000:1100].cpu().numpy()) <= 2e-6
    y2 = cd.dot(enc, 2.0 * x)
    assert torch.equal(y2, 2.0 * y)  # exact: scaling by 2 commutes with fp32 rounding
    ref = c_oracle.dot(c_oracle.encode(w, "cser"), xs[1568][:, 1500:].astype(np.float64))
    assert rel_err(y[:, 1500:].cpu().numpy(), ref) <= REL_TOL


@pytest.mark.parametrize("name,batch", [("alexnet-fc6", 64), ("vgg-fc6", 96), ("resnet-conv", 200), ("oracle", 37)])
def test_matmat_kernels_agree_bitwise(name, batch):
    """The flat entry-stream mat-mat kernel and the per-segment one compute every column in the same
    fp32 order: identical outputs (V = 1, 2, 4; full and partial column chunks; CER and CSER)."""
    from paper_1805_10692_b200._native import force_path

    w, _ = synth.make_layer(name)
    x = torch.from_numpy(np.random.default_rng(2).standard_normal((w.shape[1], batch), dtype=np.float32)).cuda()
    wt = torch.from_numpy(w).cuda()
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(wt)
        with force_path("matmat", "segment"):
            y0 = cd.dot(enc, x)
        with force_path("matmat", "flat"):
            y1 = cd.dot(enc, x)
        assert torch.equal(y0, y1), (name, encode.__name__)


@pytest.mark.parametrize("path", ["1", "2", "3", "4", "5"])
def test_u32_column_indices(kernel_path, path):
    """n > 65535 (u32 colI): every mat-vec kernel and the mat-mat kernel, integer alphabet -> bitwise."""
    kernel_path("matvec", int(path))
    rng = np.random.default_rng(31)
    m, n = 40, 70001
    w = rng.choice(np.arange(-3.0, 4.0), size=(m, n), p=[0.02, 0.03, 0.05, 0.8, 0.05, 0.03, 0.02])
    w[3] = 0.0
    x = rng.integers(-2, 3, size=(n, 5)).astype(np.float64)
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(w)
        assert enc.col_index_bits == 32
        assert np.array_equal(cd.dot(enc, x[:, 0]), w @ x[:, 0]), encode.__name__
        assert np.array_equal(cd.dot(enc, x), w @ x), encode.__name__


def test_long_rows_default_to_run_kernel_and_match_oracle():
    """Rows of >= 4096 entries take the long-row (stream) kernel by default (colI ring across rows, several
    segment batches inside one window, CER padding); integer alphabet -> bitwise, real -> 1e-5."""
    rng = np.random.default_rng(21)
    m, n = 96, 20000
    levels = np.arange(-12, 13, dtype=np.float64)
    p = np.exp(-np.abs(levels) / 3.0)
    p[12] = 4.0 * p.sum()  # zero is the mode (~70%)
    w = rng.choice(levels, size=(m, n), p=p / p.sum())
    w[17, :] = 0.0  # an empty row between long ones
    x = rng.integers(-3, 4, size=n).astype(np.float64)
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(w)
        assert enc.nnz >= 4096 * m * 0.5
        assert np.array_equal(cd.dot(enc, x), w @ x), encode.__name__
        xr = rng.standard_normal(n)
        ref = c_oracle.dot(c_oracle.encode(w, "cer" if encode is cd.encode_cer else "cser"), xr)
        assert rel_err(cd.dot(enc, xr.astype(np.float32)), ref) <= REL_TOL, encode.__name__


def test_device_draw_equals_numpy_draw():
    """synth.make_weights_device (PCG64 on the device) is bit-identical to the seeded numpy draw, for whole
    layers and for row blocks in the middle of config 5 (reached on the host with bit_generator.advance)."""
    for name in ("oracle", "alexnet-fc6", "resnet-conv"):
        cfg = synth.config(name)
        host = synth.make_weights(cfg, np.random.default_rng(0))
        assert np.array_equal(synth.make_weights_device(cfg, 0, "cuda").cpu().numpy(), host), name
    cfg = synth.config("large")
    for row0 in (0, 12345, 32700):
        rng = np.random.default_rng(0)
        rng.bit_generator.advance(row0 * cfg.n)
        host = synth.make_weights(cfg, rng, rows=40)
        dev = synth.make_weights_device(cfg, 0, "cuda", row0=row0, rows=40).cpu().numpy()
        assert np.array_equal(dev, host), row0


def test_large_config_properties():
    """Config 5 (32768^2, 256 levels) at full size: CER and CSER agree, scaling x by 2 is exact, and a
    row slice matches the oracle (size-independent checks; W drawn on the device)."""
    cfg = synth.config("large")
    w = synth.make_weights_device(cfg, 0, "cuda")
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(cfg.n, dtype=np.float32)).cuda()
    cer, cser = cd.encode_cer(w), cd.encode_cser(w)
    y_cer, y_cser = cd.dot(cer, x), cd.dot(cser, x)
    assert rel_err(y_cer.cpu().numpy(), y_cser.double().cpu().numpy()) <= REL_TOL
    assert torch.equal(cd.dot(cer, 2.0 * x), 2.0 * y_cer)
    rows = w[:64].cpu().numpy()
    del w
    ref = c_oracle.dot(c_oracle.encode(rows, "cser"), x.cpu().numpy().astype(np.float64))
    assert rel_err(y_cser[:64].cpu().numpy(), ref) <= REL_TOL


def test_background_nonzero_without_decomposition():
    # criterion-7 shaped matrices (mode != 0) encoded directly: y += bg * sum(x) in the epilogue
    for seed in range(10):
        w, x = recipes.nonzero_mode(seed)
        for encode, ref_encode in ((cd.encode_cer, numpy_port.encode_cer), (cd.encode_cser, numpy_port.encode_cser)):
            enc = encode(w)
            assert enc.background != 0.0
            assert rel_err(cd.dot(enc, x), numpy_port.dot(ref_encode(w), x)) <= REL_TOL
            xb = np.random.default_rng(seed).normal(size=(w.shape[1], 5))
            assert rel_err(cd.dot(enc, xb), numpy_port.dot(ref_encode(w), xb)) <= REL_TOL


def test_torch_api_and_determinism():
    w, xs = synth.make_layer("oracle")
    enc = cd.encode_cer(torch.from_numpy(w).cuda())
    x = torch.from_numpy(xs[1]).cuda()
    y1 = cd.dot_device(enc, x)
    y2 = cd.dot_device(enc, x)
    assert y1.dtype == torch.float32 and y1.is_cuda and y1.shape == (512,)
    assert torch.equal(y1, y2)
    y_np = cd.dot(enc, xs[1])
    assert np.array_equal(y_np, y1.cpu().numpy().astype(np.float64))
    y_t, tr = cd.dot_cer(enc, x, trace=True)
    assert torch.equal(y_t, y1) and tr.count("read", "colI") == enc.nnz
    with pytest.raises(ValueError, match="mismatch"):
        cd.dot(enc, torch.ones(5, device="cuda"))
    with pytest.raises(TypeError):
        cd.dot_cser(enc, x)


def test_host_constructed_encoding_uploads(small_cases):
    case = next(c for c in small_cases if c["name"] == "M_ones")
    g = case["cer"]
    enc = cd.CerMatrix(np.array(g["omega"]), np.array(g["colI"], dtype=np.int64), np.array(g["omegaPtr"]),
                       np.array(g["rowPtr"]), 5, 12)
    assert cd.dot(enc, np.ones(12)).tolist() == [22.0, 24.0, 17.0, 23.0, 16.0]


def test_negative_zero_and_nan_handling():
    enc = cd.encode_cer(np.array([[-0.0, -0.0, 1.0]]))
    assert np.signbit(enc.omega[0]) and enc.col_index.tolist() == [2]
    enc = cd.encode_cer(np.array([[0.0, -0.0, 0.0, 1.0, 1.0]]))  # mixed zeros are one element
    assert enc.omega.tolist() == [0.0, 1.0] and not np.signbit(enc.omega[0])
    assert enc.col_index.tolist() == [3, 4]
    ref = numpy_port.encode_cer(np.array([[np.nan, 1.0, 1.0]]))
    enc = cd.encode_cer(np.array([[np.nan, 1.0, 1.0]]))
    assert enc.col_index.tolist() == ref["colI"].tolist() and np.isnan(enc.omega[1])


def test_empty_and_degenerate():
    with pytest.raises(IndexError):
        cd.encode_cer(np.zeros((0, 4)))
    with pytest.raises(IndexError):
        cd.encode_cser(np.zeros((3, 0)))
    enc = cd.encode_cer(np.zeros((4, 5)))
    assert cd.dot(enc, np.arange(5.0)).tolist() == [0.0] * 4
    enc = cd.encode_cser(np.full((3, 7), 2.5))  # constant, background 2.5: y = 2.5 * sum(x)
    assert np.allclose(cd.dot(enc, np.arange(7.0)), 2.5 * 21.0)


def test_wide_alphabets_up_to_fast_limit():
    rng = np.random.default_rng(5)
    w = rng.integers(-1000, 1000, size=(64, 300)).astype(np.float64)  # ~1900 distinct values
    x = rng.integers(-3, 4, size=300).astype(np.float64)
    for encode, ref_encode in ((cd.encode_cer, numpy_port.encode_cer), (cd.encode_cser, numpy_port.encode_cser)):
        enc = encode(w)
        ref = ref_encode(w)
        assert digest(enc.col_index) == digest(ref["colI"])
        assert digest(enc.omega_ptr) == digest(ref["omegaPtr"])
        assert digest(enc.row_ptr) == digest(ref["rowPtr"])
        assert np.array_equal(cd.dot(enc, x), w @ x)


@pytest.mark.parametrize("path", ["tile", "window", "run", "stream", "row"])
@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6", "resnet-conv"])
def test_matvec_paths_agree_with_oracle(kernel_path, config_goldens, name, path):
    """Every mat-vec kernel (CTA-tile TMA pipeline, warp-window, run, stream and row kernels) meets the bar."""
    kernel_path("matvec", path)
    meta, ys = config_goldens
    w, _ = synth.make_layer(name)
    x1 = np.random.default_rng(1).standard_normal(w.shape[1], dtype=np.float32)
    wt = torch.from_numpy(w).cuda()
    for kind in ("cer", "cser"):
        enc = (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt)
        assert rel_err(cd.dot(enc, x1), ys[f"{name}/{kind}/b1"]) <= REL_TOL, (name, kind, path)


@pytest.mark.parametrize("path", ["1", "2", "3", "4", "5"])
def test_matvec_tile_edge_rows(kernel_path, path):
    """Empty rows, single-entry rows, a long row next to short ones, non-zero background (every kernel)."""
    kernel_path("matvec", int(path))
    rng = np.random.default_rng(9)
    w = np.zeros((300, 700))
    w[5, :] = rng.integers(1, 4, size=700)           # a dense row (700 entries, few segments)
    w[7, 3] = 2.0                                     # single entry
    w[100:300:3, ::5] = rng.integers(-3, 4, size=(67, 140))
    x = rng.integers(-4, 5, size=700).astype(np.float64)
    for bg in (None, 1.0):
        for encode in (cd.encode_cer, cd.encode_cser):
            enc = encode(w, background=bg)
            y = cd.dot(enc, x)
            assert np.array_equal(y, w @ x), (encode.__name__, bg)


@pytest.mark.parametrize("shape,distinct", [((64, 300), None), ((40, 120), 2100), ((7, 5000), 3000)])
def test_sort_path_large_alphabets(shape, distinct):
    """Alphabets beyond the on-chip tables take the sort-based conversion: still bit-exact."""
    rng = np.random.default_rng(sum(shape))
    if distinct is None:  # every value distinct (quantised-free real matrix)
        w = rng.normal(size=shape)
    else:
        w = rng.choice(rng.normal(size=distinct), size=shape)
        w[rng.random(shape) < 0.3] = 0.0
    x = rng.normal(size=shape[1])
    for bg in (None, 0.0, 12.5):
        for encode, ref_encode in ((cd.encode_cer, numpy_port.encode_cer), (cd.encode_cser, numpy_port.encode_cser)):
            enc = encode(w, background=bg)
            ref = ref_encode(w, background=bg)
            tag = (shape, distinct, bg, encode.__name__)
            assert np.array_equal(enc.omega, ref["omega"]), tag
            assert np.array_equal(enc.col_index, ref["colI"]) and enc.col_index.dtype == ref["colI"].dtype, tag
            assert np.array_equal(enc.omega_ptr, ref["omegaPtr"]) and enc.omega_ptr.dtype == ref["omegaPtr"].dtype, tag
            assert np.array_equal(enc.row_ptr, ref["rowPtr"]) and enc.row_ptr.dtype == ref["rowPtr"].dtype, tag
            if encode is cd.encode_cser:
                assert np.array_equal(enc.omega_index, ref["omegaI"]), tag
                assert enc.mode_index == ref["mode_index"], tag
            assert rel_err(cd.dot(enc, x), numpy_port.dot(ref, x)) <= REL_TOL, tag


@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6"])
def test_row_entry_index(name):
    """The derived rowEntry index equals omegaPtr[rowPtr[r]], and the dot is bitwise the same with or without it."""
    w, _ = synth.make_layer(name)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal(w.shape[1], dtype=np.float32)).cuda()
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(torch.from_numpy(w).cuda())
        dev = enc.device_encoding()
        re = dev.to_host("rowEntry")
        assert np.array_equal(re, enc.omega_ptr.astype(np.int64)[enc.row_ptr.astype(np.int64)])
        assert dev.struct().row_entry
        for path in ("1", "2", "4", "5"):
            from paper_1805_10692_b200._native import force_path

            with force_path("matvec", int(path)):
                y_re = cd.dot_device(enc, x).cpu().numpy()
                dev._row_entry_ready = False
                dev._struct = None
                assert not dev.struct().row_entry
                y_plain = cd.dot_device(enc, x).cpu().numpy()
                dev._row_entry_ready = True
                dev._struct = None
            assert np.array_equal(y_re, y_plain), (name, encode.__name__, path)


@pytest.mark.parametrize("name", ["alexnet-fc6", "vgg-fc6"])
def test_host_buffer_path(config_goldens, name):
    """The host-buffer path (pinned staging, one C call: H2D, kernel, D2H, sync) equals the device path
    bitwise, meets the oracle bar, and survives repeated calls with alternating matrices."""
    meta, ys = config_goldens
    w, _ = synth.make_layer(name)
    x1 = np.random.default_rng(1).standard_normal(w.shape[1], dtype=np.float32)
    wt = torch.from_numpy(w).cuda()
    encs = {kind: (cd.encode_cer if kind == "cer" else cd.encode_cser)(wt) for kind in ("cer", "cser")}
    xd = torch.from_numpy(x1).cuda()
    for rep in range(3):
        for kind, enc in encs.items():
            y_host = cd.dot(enc, x1)
            y_dev = cd.dot_device(enc, xd).cpu().numpy().astype(np.float64)
            assert np.array_equal(y_host, y_dev), (name, kind, rep)
            assert rel_err(y_host, ys[f"{name}/{kind}/b1"]) <= REL_TOL, (name, kind)


def test_host_buffer_raw_abi_pageable_and_pinned():
    """cerdot_dot_host through ctypes with pageable numpy buffers and with pinned buffers."""
    from paper_1805_10692_b200 import _native
    w, _ = synth.make_layer("alexnet-fc6")
    enc = cd.encode_cer(torch.from_numpy(w).cuda())
    st = enc.device_encoding().struct()
    L = _native.lib()
    x = np.random.default_rng(5).standard_normal(w.shape[1]).astype(np.float32)
    ws_bytes = L.cerdot_dot_host_workspace_bytes(st, 1)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    y_ref = cd.dot_device(enc, torch.from_numpy(x).cuda()).cpu().numpy()
    stream = torch.cuda.current_stream().cuda_stream
    y_page = np.empty(w.shape[0], dtype=np.float32)
    _native.check(L.cerdot_dot_host(st, x.ctypes.data, 1, 1, y_page.ctypes.data, 1, ws.data_ptr(), ws_bytes, stream))
    assert np.array_equal(y_page, y_ref)
    px = torch.from_numpy(x).pin_memory()
    py = torch.empty(w.shape[0], dtype=torch.float32).pin_memory()
    for _ in range(3):
        py.zero_()
        _native.check(L.cerdot_dot_host(st, px.data_ptr(), 1, 1, py.data_ptr(), 1, ws.data_ptr(), ws_bytes, stream))
        assert np.array_equal(py.numpy(), y_ref)


@pytest.mark.parametrize("name,batch", [("alexnet-fc6", 1), ("resnet-conv", 1), ("alexnet-fc6", 16),
                                        ("resnet-conv", 40)])
def test_fused_peer_exchange_emulated_ranks(name, batch):
    """cerdot_dot_peers, ranks emulated on one GPU (each rank's kernel runs alone; no cross-rank wait):
    rank r's shard writes its rows into its own buffer and, from the epilogue, into every other rank's
    buffer.  Afterwards all buffers hold the full product (identical), within the bar of the oracle."""
    from paper_1805_10692_b200 import shard

    w, _ = synth.make_layer(name)
    rng = np.random.default_rng(4)
    xn = rng.standard_normal((w.shape[1], batch) if batch > 1 else w.shape[1], dtype=np.float32)
    x = torch.from_numpy(xn).cuda()
    ranks = 3
    for kind in ("cer", "cser"):
        full = (cd.encode_cer if kind == "cer" else cd.encode_cser)(torch.from_numpy(w).cuda())
        bounds = shard.plan_rows(full, ranks)
        shape = (full.m,) if batch == 1 else (full.m, batch)
        bufs = [torch.full(shape, float("nan"), device="cuda") for _ in range(ranks)]
        for r in range(ranks):
            local = shard.slice_rows(full, bounds[r], bounds[r + 1])
            peers = torch.tensor([b.data_ptr() for p, b in enumerate(bufs) if p != r], dtype=torch.int64,
                                 device="cuda")
            off = bounds[r] * (1 if batch == 1 else batch)
            cd.dot_device(local, x, out=bufs[r][bounds[r]:bounds[r + 1]], peers=peers, peer_offset=off)
        torch.cuda.synchronize()
        for b in bufs[1:]:
            assert torch.equal(b, bufs[0]), (name, kind)
        ref = c_oracle.dot(c_oracle.encode(w, kind), xn.astype(np.float64))
        assert rel_err(bufs[0].cpu().numpy(), ref) <= REL_TOL, (name, kind)


def test_peer_row_sharded_dot_single_rank():
    """PeerRowShardedDot end to end (symmetric memory, barrier) in a one-rank NCCL group."""
    import os
    import socket

    import torch.distributed as dist

    from paper_1805_10692_b200 import shard

    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        w, xs = synth.make_layer("alexnet-fc6")
        enc = cd.encode_cer(torch.from_numpy(w).cuda())
        op = shard.PeerRowShardedDot(enc, [enc.m], batch=1)
        x = torch.from_numpy(xs[1]).cuda()
        y = op(x)
        torch.cuda.synchronize()
        assert torch.equal(y, cd.dot_device(enc, x))
    finally:
        dist.destroy_process_group()


def test_device_validate_and_decode_match_reference(validate_cases):
    """cd.validate (cerdot_validate on the device) raises the reference's FormatError -- same array,
    offset and reason -- for all 1395 corrupted encodings of tests/golden/validate_cases.json, and
    cd.decode reproduces the reference's dense matrix (sha256) for every accepted one."""
    import hashlib

    from conftest import validate_case_arrays

    bases = validate_cases["bases"]
    for case in validate_cases["cases"]:
        e = validate_case_arrays(bases, case)
        if e["kind"] == "cer":
            enc = cd.CerMatrix(e["omega"], e["colI"], e["omegaPtr"], e["rowPtr"], e["m"], e["n"])
        else:
            enc = cd.CserMatrix(e["omega"], e["colI"], e["omegaI"], e["omegaPtr"], e["rowPtr"], e["m"], e["n"],
                                mode_index=e["mode_index"])
        if case["error"]:
            with pytest.raises(cd.FormatError) as err:
                cd.validate(enc)
            got = [err.value.array, err.value.offset, err.value.reason]
            assert got == case["error"], (case, got)
        else:
            cd.validate(enc)
            dense = cd.decode(enc).values
            assert hashlib.sha256(np.ascontiguousarray(dense).tobytes()).hexdigest() == case["decode_sha256"], case


@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6", "resnet-conv"])
def test_device_decode_round_trip_configs(name):
    """Encoder output validates and decodes back to W exactly (the reference's TestRoundTrip), device-resident."""
    w, _ = synth.make_layer(name)
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(torch.from_numpy(w).cuda())
        cd.validate(enc)
        assert np.array_equal(cd.decode(enc).values, w.astype(np.float64)), (name, encode.__name__)


def test_corruption_fuzz_every_single_entry():
    """The reference's TestCorruptionFuzz (tests/test_formats.py:214-235) on the device: EVERY
    (position, value) corruption of M's pointer and omegaI arrays; >= 99% rejected, and each outcome
    identical to the pinned oracle's."""
    from oracle import numpy_port

    w = np.array([[0, 3, 0, 2, 4, 0, 0, 2, 3, 4, 0, 4], [4, 4, 0, 0, 0, 4, 0, 0, 4, 4, 0, 4],
                  [4, 0, 3, 4, 0, 0, 0, 4, 0, 2, 0, 0], [0, 0, 0, 4, 4, 4, 0, 3, 4, 4, 0, 0],
                  [0, 4, 4, 0, 0, 4, 0, 4, 0, 0, 0, 0]], dtype=float)
    for kind in ("cer", "cser"):
        base = (numpy_port.encode_cer if kind == "cer" else numpy_port.encode_cser)(w)
        names = ["omegaPtr", "rowPtr"] + (["omegaI"] if kind == "cser" else [])
        for name in names:
            arr = np.asarray(base[name])
            total = accepted = 0
            for pos in range(arr.size):
                for value in range(1 << (arr.dtype.itemsize * 8)):
                    if value == arr[pos]:
                        continue
                    e = dict(base)
                    e[name] = arr.copy()
                    e[name][pos] = value
                    if kind == "cer":
                        enc = cd.CerMatrix(e["omega"], e["colI"], e["omegaPtr"], e["rowPtr"], e["m"], e["n"])
                    else:
                        enc = cd.CserMatrix(e["omega"], e["colI"], e["omegaI"], e["omegaPtr"], e["rowPtr"], e["m"],
                                            e["n"], mode_index=e["mode_index"])
                    want = numpy_port.validate(e)
                    total += 1
                    try:
                        cd.validate(enc)
                        got = None
                    except cd.FormatError as err:
                        got = (err.array, err.offset, err.reason)
                    assert got == want, (kind, name, pos, value, got, want)
                    accepted += got is None
            assert 1.0 - accepted / total >= 0.99, (kind, name, accepted, total)


@pytest.mark.parametrize("name", ["oracle", "alexnet-fc6", "resnet-conv"])
def test_device_trace_counts_match_host_trace(name):
    """trace_of on a device-resident encoding (cerdot_trace_counts) == trace_of on the same arrays held
    on the host (the reference's analytic trace, kernels.py:175-234), for 1 and 7 columns."""
    w, _ = synth.make_layer(name)
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(torch.from_numpy(w).cuda())
        if isinstance(enc, cd.CerMatrix):
            host = cd.CerMatrix(enc.omega, enc.col_index, enc.omega_ptr, enc.row_ptr, enc.m, enc.n, enc.element_bits)
        else:
            host = cd.CserMatrix(enc.omega, enc.col_index, enc.omega_index, enc.omega_ptr, enc.row_ptr, enc.m, enc.n,
                                 enc.element_bits, enc.mode_index)
        for cols in (1, 7):
            assert cd.trace_of(enc, columns=cols).counts == cd.trace_of(host, columns=cols).counts, (name, cols)


def test_randomized_round_trip_and_dot():
    """The reference's TestRoundTrip shape (random low-entropy matrices, tests/test_formats.py:142-150)
    through the whole device path: encode (bit-exact vs the oracle), validate, decode == W, and the
    mat-vec / mat-mat through every kernel path against the oracle (integer alphabets: bitwise)."""
    import os

    from paper_1805_10692_b200._native import force_path

    rng = np.random.default_rng(int(os.environ.get("CERDOT_FUZZ_SEED", "1805")))
    for trial in range(int(os.environ.get("CERDOT_FUZZ_TRIALS", "60"))):
        m, n, kk = int(rng.integers(1, 70)), int(rng.integers(1, 400)), int(rng.integers(1, 9))
        elems = np.unique(rng.integers(-5, 6, size=kk)).astype(float)
        wts = rng.random(elems.size) + 0.1
        w = rng.choice(elems, size=(m, n), p=wts / wts.sum())
        x = rng.integers(-3, 4, size=(n, 3)).astype(np.float64)
        for kind, encode in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
            enc = encode(cd.DenseMatrix(w))
            ref = (numpy_port.encode_cer if kind == "cer" else numpy_port.encode_cser)(w)
            assert np.array_equal(enc.col_index, ref["colI"]) and np.array_equal(enc.omega_ptr, ref["omegaPtr"])
            assert np.array_equal(enc.row_ptr, ref["rowPtr"]) and np.array_equal(enc.omega, ref["omega"])
            cd.validate(enc)
            assert np.array_equal(cd.decode(enc).values, w), (trial, kind)
            assert np.array_equal(cd.dot(enc, x), w @ x), (trial, kind)
            assert np.array_equal(cd.dot(enc, x[:, 0]), w @ x[:, 0]), (trial, kind)
            for path in ("window", "tile", "run", "stream", "row"):
                with force_path("matvec", path):
                    assert np.array_equal(cd.dot(enc, x[:, 1]), w @ x[:, 1]), (trial, kind, path)


def test_device_row_slices_equal_host_slices():
    """shard.slice_rows_device (bench.py's N>1 shards of the global encoding) == shard.slice_rows, array by
    array, and the blocks' products concatenate to the full product within the bar (not bitwise: a block's
    kernel choice and window alignment follow its own row count and rebased entry offsets)."""
    from paper_1805_10692_b200 import shard

    w, xs = synth.make_layer("alexnet-fc6")
    x = torch.from_numpy(xs[1]).cuda()
    for encode in (cd.encode_cer, cd.encode_cser):
        full = encode(torch.from_numpy(w).cuda())
        y_full = cd.dot(full, x)
        for parts in (2, 4, 8):
            bounds = shard.plan_rows(full, parts)
            ys = []
            for a, b in zip(bounds[:-1], bounds[1:]):
                d, h = shard.slice_rows_device(full, a, b), shard.slice_rows(full, a, b)
                for f in ("col_index", "omega_ptr", "row_ptr") + (("omega_index",) if encode is cd.encode_cser else ()):
                    assert np.array_equal(getattr(d, f), getattr(h, f)), (f, a, b)
                ys.append(cd.dot(d, x))
            assert rel_err(torch.cat(ys).cpu().numpy(), y_full.double().cpu().numpy()) <= REL_TOL, (encode.__name__,
                                                                                                    parts)


def test_untrusted_host_encoding_is_validated_before_the_kernels():
    """A host-constructed encoding with an out-of-range column index raises FormatError at its first
    device use (it would otherwise index x out of bounds inside the kernels); a valid one runs."""
    w, xs = synth.make_layer("oracle")
    ref = numpy_port.encode_cer(w)
    good = cd.CerMatrix(ref["omega"], ref["colI"], ref["omegaPtr"], ref["rowPtr"], ref["m"], ref["n"])
    assert rel_err(cd.dot(good, xs[1]), numpy_port.dot(ref, xs[1])) <= REL_TOL
    col = np.array(ref["colI"]).copy()
    col[5] = ref["n"] + 7
    bad = cd.CerMatrix(ref["omega"], col, ref["omegaPtr"], ref["rowPtr"], ref["m"], ref["n"])
    with pytest.raises(cd.FormatError):
        cd.dot(bad, xs[1])
    torch.cuda.synchronize()  # the context is intact


def test_encode_pair_equals_separate_encodes():
    """encode_pair (one shared plan, two fills) == encode_cer and encode_cser array by array: a sparse fc
    layer (compacting fill), a dense-ish one, an alphabet on the sort path, an explicit background."""
    rng = np.random.default_rng(77)
    big = rng.choice(rng.normal(size=3000), size=(40, 500))
    big[rng.random(big.shape) < 0.4] = 0.0
    cases = [(synth.make_layer("oracle")[0], None), (synth.make_layer("resnet-conv")[0], None), (big, None),
             (synth.make_layer("oracle")[0], 0.25)]
    for w, bg in cases:
        wt = torch.from_numpy(w).cuda()
        cer, cser = cd.encode_pair(wt, background=bg)
        for got, want in ((cer, cd.encode_cer(wt, background=bg)), (cser, cd.encode_cser(wt, background=bg))):
            assert type(got) is type(want)
            for name in ("omega", "col_index", "omega_ptr", "row_ptr"):
                assert np.array_equal(getattr(got, name), getattr(want, name)), (w.shape, bg, name)
            if isinstance(got, cd.CserMatrix):
                assert np.array_equal(got.omega_index, want.omega_index) and got.mode_index == want.mode_index
        x = torch.from_numpy(rng.standard_normal(w.shape[1], dtype=np.float32)).cuda()
        assert torch.equal(cd.dot(cer, x), cd.dot(cd.encode_cer(wt, background=bg), x))


@pytest.mark.parametrize("name", ["alexnet-fc6", "oracle"])
def test_row_kernel_bitwise_equals_window_kernel(name):
    """The one-row-per-warp kernel runs the window kernel's single-window arithmetic: identical bits, on the
    configs' own x, an all-positive x and a misaligned x view; and it is the automatic choice for AlexNet fc6."""
    from paper_1805_10692_b200._native import force_path

    w, xs = synth.make_layer(name)
    rng = np.random.default_rng(8)
    wt = torch.from_numpy(w).cuda()
    pad = torch.zeros(w.shape[1] + 1, device="cuda")
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(wt)
        for xv in (xs[1].reshape(-1), np.abs(rng.standard_normal(w.shape[1], dtype=np.float32))):
            x = torch.from_numpy(xv).cuda()
            with force_path("matvec", "window"):
                y_win = cd.dot_device(enc, x)
            with force_path("matvec", "row"):
                y_row = cd.dot_device(enc, x)
                pad[1:] = x
                y_mis = cd.dot_device(enc, pad[1:])  # 4 B-aligned x: cooperative staging
            assert torch.equal(y_win, y_row) and torch.equal(y_win, y_mis), (name, encode.__name__)
            if name == "alexnet-fc6":
                assert torch.equal(cd.dot_device(enc, x), y_row)


@pytest.mark.parametrize("levels", [9, 700])
def test_stream_kernel_alphabets_modes_and_row_shapes(levels):
    """The stream kernel on long rows with a small (u8 flags) and a wide (u16 flags) alphabet, a CSER mode in
    the middle of the alphabet, empty rows, a row of one segment, rows ending exactly at a window boundary:
    integer data -> bitwise w @ x; the same through the run and window kernels."""
    from paper_1805_10692_b200._native import force_path

    rng = np.random.default_rng(levels)
    m, n = 37, 6000
    vals = np.arange(-(levels // 2), levels - levels // 2).astype(np.float64)
    p = rng.random(levels) + 0.05
    p[levels // 2] += 0.6 * p.sum()  # a dominant value (0) in the middle of the sorted alphabet
    w = rng.choice(vals, size=(m, n), p=p / p.sum())
    w[3] = 0.0                     # empty row
    w[5] = 4.0                     # one segment of n entries (23 full windows + a tail)
    w[7, :] = 0.0
    w[7, :2048] = 2.0              # ends exactly at a window boundary
    w[9, 100:101] = -1.0
    x = rng.integers(-2, 3, size=n).astype(np.float64)
    for bg in (None, 1.0):
        for encode in (cd.encode_cer, cd.encode_cser):
            enc = encode(w, background=bg)
            want = w @ x
            for path in ("stream", "run", "window"):
                with force_path("matvec", path):
                    assert np.array_equal(cd.dot(enc, x), want), (levels, bg, encode.__name__, path)
            for nt in (768, 896):
                with force_path("matvec", "stream"), force_path("matvec_nt", nt):
                    assert np.array_equal(cd.dot(enc, x), want), (levels, bg, encode.__name__, nt)


@pytest.mark.parametrize("path,m,n", [("stream", 150, 6000), ("row", 5000, 600), ("row", 90, 600)])
def test_coalesced_peer_stores_stream_and_row_kernels(path, m, n):
    """The peers instances of the stream kernel (32 results per warp in one store) and of the row kernel (a
    CTA's contiguous rows staged, stored together): three emulated ranks, integer data -> every rank's
    buffer holds exactly w @ x (uneven shards, rows that end mid-group, empty rows)."""
    from paper_1805_10692_b200 import shard
    from paper_1805_10692_b200._native import force_path

    rng = np.random.default_rng(m + n)
    w = rng.choice(np.arange(-3.0, 4.0), size=(m, n), p=[0.03, 0.04, 0.05, 0.76, 0.05, 0.04, 0.03])
    w[1] = 0.0
    w[m - 1] = 0.0
    x = rng.integers(-2, 3, size=n).astype(np.float64)
    xt = torch.from_numpy(x.astype(np.float32)).cuda()
    want = torch.from_numpy((w @ x).astype(np.float32)).cuda()
    ranks = 3
    for encode in (cd.encode_cer, cd.encode_cser):
        full = encode(w)
        bounds = [0, m // 5, m // 5 + m // 2, m]
        bufs = [torch.full((m,), float("nan"), device="cuda") for _ in range(ranks)]
        with force_path("matvec", path):
            for r in range(ranks):
                local = shard.slice_rows(full, bounds[r], bounds[r + 1])
                peers = torch.tensor([b.data_ptr() for q, b in enumerate(bufs) if q != r], dtype=torch.int64,
                                     device="cuda")
                cd.dot_device(local, xt, out=bufs[r][bounds[r]:bounds[r + 1]], peers=peers, peer_offset=bounds[r])
        torch.cuda.synchronize()
        for b in bufs:
            assert torch.equal(b, want), (path, encode.__name__)
