"""GPU: the TMA-staged mat-mat over the column-tiled view (csrc/tileview.cu).

* the view itself (tile_ptr / tile_rec) is bit-exact against a numpy restatement of its definition
  (every segment of kernels.py:283-301 split at the X-tile boundaries; colI ascending inside a segment,
  formats.py:220);
* the mat-mat meets the 1e-5 bar against the C oracle (the reference's loop order, float64) on configs
  1-4 at their BASELINE batches -- config 4 at B=1568 on every column, in column chunks -- and is bitwise
  on integer alphabets;
* edge cases: empty rows, a dense row, a row inside one tile, n and B not multiples of the tile sizes,
  padded row strides of X, u8 / u32 column indices, CER and CSER, non-zero background;
* deterministic (two calls bitwise equal) and within the bar of the flat L2-gather kernel.
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


def tile_view_np(enc, nt: int):
    """numpy restatement of the view: records tile-major, then row, then the encoding's entry order; each
    record = (its X row inside the tile | matrix row (low 12 bits) << 9 | row end << 30 | fragment end << 31,
    fp32 segment value)."""
    rp = enc.row_ptr.astype(np.int64)
    op = enc.omega_ptr.astype(np.int64)
    col = enc.col_index.astype(np.int64)
    m, n = enc.m, enc.n
    nseg = op.size - 1
    seg_row = np.repeat(np.arange(m), np.diff(rp))
    if isinstance(enc, cd.CserMatrix):
        k = enc.omega_index.astype(np.int64)
        bg = float(enc.omega[enc.mode_index])
    else:
        k = np.arange(nseg) - rp[seg_row] + 1
        bg = float(enc.omega[0])
    v = (enc.omega[k] - bg).astype(np.float32)
    sizes = np.diff(op)
    ent_seg = np.repeat(np.arange(nseg), sizes)
    ent_row = seg_row[ent_seg]
    tile = col // nt
    nxt_same_seg = np.zeros(col.size, dtype=bool)
    nxt_same_seg[:-1] = ent_seg[1:] == ent_seg[:-1]
    nxt_tile = np.empty_like(tile)
    nxt_tile[:-1] = tile[1:]
    nxt_tile[-1:] = -1
    end = ~(nxt_same_seg & (nxt_tile == tile))
    order = np.lexsort((np.arange(col.size), ent_row, tile))
    rec = np.empty((col.size, 2), dtype=np.uint32)
    # row end: the last record of its (row, tile) list, i.e. the next record in view order changes (tile, row)
    o_tile, o_row = tile[order], ent_row[order]
    row_end = np.ones(col.size, dtype=bool)
    row_end[:-1] = (o_tile[1:] != o_tile[:-1]) | (o_row[1:] != o_row[:-1])
    rec[:, 0] = ((col - tile * nt) | ((ent_row & 0xFFF) << 9) | (end.astype(np.int64) << 31))[order] | (
        row_end.astype(np.int64) << 30)
    rec[:, 1] = v[ent_seg].view(np.uint32)[order]
    tiles = -(-n // nt)
    cnt = np.zeros((tiles, m), dtype=np.int64)
    np.add.at(cnt, (tile, ent_row), 1)
    tptr = np.concatenate(([0], np.cumsum(cnt.ravel()))).astype(np.uint32)
    return tptr, rec


def _view(enc, batch):
    dev = enc.device_encoding()
    with force_path("matmat", "tiled"):
        s = dev.tile_struct(batch, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    nt = int(s.tile_rows)
    assert nt > 0
    tptr, rec = dev._tile_views[nt][:2]
    return nt, tptr.cpu().numpy().view(np.uint32), rec.cpu().numpy().view(np.uint32).reshape(-1, 2)


@pytest.mark.parametrize("name,batch", [("oracle", 37), ("oracle", 64), ("oracle", 200), ("alexnet-fc6", 64),
                                        ("resnet-conv", 1568)])
def test_tile_view_bit_exact(name, batch):
    w, _ = synth.make_layer(name)
    wt = torch.from_numpy(w).cuda()
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(wt)
        nt, tptr, rec = _view(enc, batch)
        tptr_ref, rec_ref = tile_view_np(enc, nt)
        assert np.array_equal(tptr, tptr_ref), (name, encode.__name__)
        assert np.array_equal(rec[: enc.nnz], rec_ref), (name, encode.__name__)


def _tiled(enc, x, path="tiled"):
    with force_path("matmat", path):
        return cd.dot(enc, x)


PATHS = ("tiled", "tiled_frag")  # per-entry fma / sum-then-multiply per segment fragment


@pytest.mark.parametrize("name,batch", [("oracle", 37), ("oracle", 64), ("oracle", 200), ("alexnet-fc6", 64),
                                        ("vgg-fc6", 128)])
def test_tiled_matmat_vs_oracle(config_goldens, name, batch):
    """Configs 1-3 at their BASELINE batches (and partial column blocks) on every row and column."""
    w, xs = synth.make_layer(name)
    x = xs[batch] if batch in xs else synth.make_inputs(synth.config(name), np.random.default_rng(5), batch)
    xt = torch.from_numpy(x).cuda()
    wt = torch.from_numpy(w).cuda()
    for kind, encode in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
        enc = encode(wt)
        ref = c_oracle.dot(c_oracle.encode(w, kind), x.astype(np.float64))
        for path in PATHS:
            y = _tiled(enc, xt, path)
            assert enc.device_encoding()._tile_views, "the tiled path did not build a view"
            err = rel_err(y.cpu().numpy(), ref)
            assert err <= REL_TOL, (name, kind, batch, path, err)
            assert torch.equal(y, _tiled(enc, xt, path))  # deterministic


def test_resnet_conv_full_batch_every_column():
    """Config 4 (mode 0.01 background, 40% zeros) at B=1568: every column against the oracle, in chunks."""
    cfg = synth.config("resnet-conv")
    w, xs = synth.make_layer(cfg)
    x = xs[1568]
    wt = torch.from_numpy(w).cuda()
    for kind, encode in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
        enc = encode(wt)
        ys = {path: _tiled(enc, torch.from_numpy(x).cuda(), path).cpu().numpy() for path in PATHS}
        ref_enc = c_oracle.encode(w, kind)
        worst = dict.fromkeys(PATHS, 0.0)
        for c0 in range(0, 1568, 392):  # column chunks of the oracle are bitwise a single call
            ref = c_oracle.dot(ref_enc, x[:, c0:c0 + 392].astype(np.float64))
            for path in PATHS:
                worst[path] = max(worst[path], rel_err(ys[path][:, c0:c0 + 392], ref))
        assert max(worst.values()) <= REL_TOL, (kind, worst)


def test_tiled_edge_rows_integer_bitwise():
    """Empty rows, a dense row, a row within one tile, single entries; integer data -> bitwise w @ x."""
    rng = np.random.default_rng(11)
    m, n = 700, 1500  # n not a multiple of any tile height
    w = np.zeros((m, n))
    w[5, :] = rng.integers(1, 4, size=n)
    w[7, 3] = 2.0
    w[9, 600:640] = rng.integers(-2, 3, size=40)
    w[100:700:3, ::5] = rng.integers(-3, 4, size=(200, 300))
    for batch in (2, 33, 64, 100, 260):
        x = rng.integers(-4, 5, size=(n, batch)).astype(np.float64)
        for bg in (None, 1.0):
            for encode in (cd.encode_cer, cd.encode_cser):
                enc = encode(w, background=bg)
                for path in PATHS:
                    y = _tiled(enc, torch.from_numpy(x.astype(np.float32)).cuda(), path).cpu().numpy()
                    assert np.array_equal(y, w @ x), (batch, bg, encode.__name__, path)


def test_tiled_padded_row_stride_and_fallback():
    """X with a padded row stride (multiple of 4: TMA) and an odd one (falls back to the flat kernel)."""
    w, _ = synth.make_layer("oracle")
    rng = np.random.default_rng(4)
    base = torch.from_numpy(rng.standard_normal((w.shape[1], 72), dtype=np.float32)).cuda()
    enc = cd.encode_cer(torch.from_numpy(w).cuda())
    ref = c_oracle.dot(c_oracle.encode(w, "cer"), base[:, :64].cpu().numpy().astype(np.float64))
    y_pad = _tiled(enc, base[:, :64])       # ldx = 72
    assert rel_err(y_pad.cpu().numpy(), ref) <= REL_TOL
    odd = torch.from_numpy(rng.standard_normal((w.shape[1], 67), dtype=np.float32)).cuda()
    y_odd = _tiled(enc, odd[:, :64])        # ldx = 67: not TMA-legal, flat kernel
    ref_odd = c_oracle.dot(c_oracle.encode(w, "cer"), odd[:, :64].cpu().numpy().astype(np.float64))
    assert rel_err(y_odd.cpu().numpy(), ref_odd) <= REL_TOL


@pytest.mark.parametrize("n", [200, 70001])
def test_tiled_u8_and_u32_columns(n):
    """colI of 8 bits (n <= 256) and 32 bits (n > 65535): integer alphabet -> bitwise."""
    rng = np.random.default_rng(n)
    m = 60
    w = rng.choice(np.arange(-3.0, 4.0), size=(m, n), p=[0.02, 0.03, 0.05, 0.8, 0.05, 0.03, 0.02])
    w[3] = 0.0
    x = rng.integers(-2, 3, size=(n, 40)).astype(np.float64)
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(w)
        assert enc.col_index_bits == (8 if n <= 256 else 32)
        for path in PATHS:
            y = _tiled(enc, torch.from_numpy(x.astype(np.float32)).cuda(), path).cpu().numpy()
            assert np.array_equal(y, w @ x), (encode.__name__, path)


@pytest.mark.parametrize("name,batch", [("alexnet-fc6", 64), ("resnet-conv", 200)])
def test_tiled_and_flat_agree(name, batch):
    w, _ = synth.make_layer(name)
    x = torch.from_numpy(np.random.default_rng(2).standard_normal((w.shape[1], batch), dtype=np.float32)).cuda()
    for encode in (cd.encode_cer, cd.encode_cser):
        enc = encode(torch.from_numpy(w).cuda())
        with force_path("matmat", "flat"):
            y_flat = cd.dot(enc, x).cpu().numpy()
        y_tiled = _tiled(enc, x).cpu().numpy()
        assert rel_err(y_tiled, y_flat) <= 2 * REL_TOL


def test_tiled_skewed_rows():
    """Power-law row lengths (a few dense rows, many near-empty ones): the entry-balanced row split per warp,
    rows longer than a warp's 32-row pointer window, and empty (row, tile) lists, against the oracle."""
    rng = np.random.default_rng(21)
    m, n = 3000, 2500
    dens = np.clip(rng.pareto(1.2, size=m) * 0.01, 0.0, 1.0)
    dens[rng.choice(m, 40, replace=False)] = 0.0
    levels = np.array([-0.3, -0.1, 0.2, 0.5, 1.5])
    w = np.where(rng.random((m, n)) < dens[:, None], levels[rng.integers(0, 5, size=(m, n))], 0.0)
    x = rng.standard_normal((n, 96)).astype(np.float32)
    for kind, encode in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
        enc = encode(w)
        ref = c_oracle.dot(c_oracle.encode(w, kind), x.astype(np.float64))
        for path in PATHS + ("flat",):
            y = _tiled(enc, torch.from_numpy(x).cuda(), path).cpu().numpy()
            assert rel_err(y, ref) <= REL_TOL, (kind, path)


def test_capture_before_the_view_exists_uses_the_flat_kernel():
    """A first batched call inside a CUDA-graph capture does not capture the tile-view build: the replay
    runs the flat kernel and gives the right answer; after an eager call, capture uses the tiled kernel."""
    w, _ = synth.make_layer("resnet-conv")
    x = torch.from_numpy(np.random.default_rng(8).standard_normal((w.shape[1], 96), dtype=np.float32)).cuda()
    enc = cd.encode_cer(torch.from_numpy(w).cuda())
    ref = c_oracle.dot(c_oracle.encode(w, "cer"), x.cpu().numpy().astype(np.float64))
    for eager_first in (False, True):
        if eager_first:
            cd.dot_device(enc, x)
            assert enc.device_encoding()._tile_views
        y = torch.empty((w.shape[0], 96), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            cd.dot_device(enc, x, out=y)
        g.replay()
        torch.cuda.synchronize()
        assert bool(enc.device_encoding()._tile_views) == eager_first
        assert rel_err(y.cpu().numpy(), ref) <= REL_TOL


@pytest.mark.parametrize("nt", [128, 256])
@pytest.mark.parametrize("split", [1, 2, 4, 8])
def test_tile_split_and_wide_tiles_integer_bitwise(nt, split):
    """The X tiles of a row block split over `split` CTAs (partial products added in split order by
    k_tv_reduce) and 256-row tiles: integer data -> bitwise w @ x, with and without a background, at a
    batch with a partial column block; the view of either tile height is bit-exact."""
    rng = np.random.default_rng(100 * nt + split)
    m, n = 333, 2100  # 17 / 9 tiles: uneven splits, a short last tile
    w = rng.choice(np.arange(-3.0, 4.0), size=(m, n), p=[0.03, 0.04, 0.05, 0.76, 0.05, 0.04, 0.03])
    w[4] = 0.0
    w[9, 1000:1300] = 2.0
    for batch in (40, 72):
        x = rng.integers(-3, 4, size=(n, batch)).astype(np.float64)
        xt = torch.from_numpy(x.astype(np.float32)).cuda()
        for bg in (None, 1.0):
            for encode in (cd.encode_cer, cd.encode_cser):
                enc = encode(w, background=bg)
                with force_path("matmat_tile", nt), force_path("matmat_split", split):
                    for path in PATHS:
                        y = _tiled(enc, xt, path).cpu().numpy()
                        assert np.array_equal(y, w @ x), (nt, split, batch, bg, encode.__name__, path)
                    vnt, tptr, rec = _view(enc, batch)
                assert vnt == nt
                tptr_ref, rec_ref = tile_view_np(enc, nt)
                assert np.array_equal(tptr, tptr_ref) and np.array_equal(rec[: enc.nnz], rec_ref)


def test_alexnet_auto_path_is_wide_tiles_with_split(config_goldens):
    """Config 2 at B=64 takes the tiled kernel automatically (256-row tiles, tiles split over CTAs) and meets the bar."""
    w, xs = synth.make_layer("alexnet-fc6")
    xt = torch.from_numpy(xs[64]).cuda()
    for kind, encode in (("cer", cd.encode_cer), ("cser", cd.encode_cser)):
        enc = encode(torch.from_numpy(w).cuda())
        y = cd.dot(enc, xt)
        assert 256 in enc.device_encoding()._tile_views, "the automatic path did not build the 256-row view"
        ref = c_oracle.dot(c_oracle.encode(w, kind), xs[64].astype(np.float64))
        assert rel_err(y.cpu().numpy(), ref) <= REL_TOL, kind
        assert torch.equal(y, cd.dot(enc, xt))
