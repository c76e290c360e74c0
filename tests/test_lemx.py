"""LEMX containers (io.py:177-278): reference-written files parse to the reference's arrays, load into
HBM, validate, and write back byte for byte; malformed files raise the reference's IoFormatError codes."""

import json
import os

import numpy as np
import pytest

import paper_1805_10692_b200 as cd
from paper_1805_10692_b200 import io as lemx

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lemx_files.json")


@pytest.fixture(scope="module")
def lemx_golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_header_parse_matches_reference_files(lemx_golden):
    for rec in lemx_golden["files"]:
        raw = bytes.fromhex(rec["hex"])
        h = lemx._parse(raw, "golden")
        assert (h["kind"], h["m"], h["n"], h["ebits"]) == (rec["kind"], rec["m"], rec["n"], rec["element_bits"])
        assert (h["k"], h["nnz"], h["segs"]) == (len(rec["omega"]), len(rec["colI"]), len(rec["omegaPtr"]) - 1)
        assert len(raw) == lemx.header_bytes(rec["kind"]) + sum(nb for _, nb in h["spans"].values())
        col_off, col_nb = h["spans"]["colI"]
        cols = np.frombuffer(raw, dtype=lemx._index_dtype(h["widths"]["colI"]), count=len(rec["colI"]), offset=col_off)
        assert cols.tolist() == rec["colI"]


def test_malformed_files_raise_reference_codes(lemx_golden, tmp_path):
    for e in lemx_golden["errors"]:
        raw = bytes.fromhex(e["hex"])
        with pytest.raises(lemx.IoFormatError) as err:
            lemx._parse(raw, "x")
        # the reference raises struct.error (not IoFormatError) on a header shorter than its fixed fields
        want = "payload-mismatch" if e["code"] == "error" else e["code"]
        assert err.value.code == want, e["label"]


@pytest.mark.gpu
def test_read_write_round_trip_on_device(lemx_golden, tmp_path):
    torch = pytest.importorskip("torch")
    path = str(tmp_path / "m.lemx")
    out = str(tmp_path / "w.lemx")
    for rec in lemx_golden["files"]:
        raw = bytes.fromhex(rec["hex"])
        open(path, "wb").write(raw)
        enc = cd.read_matrix(path)
        assert enc.device_encoding().device.type == "cuda"
        assert enc.omega.tolist() == rec["omega"]
        assert enc.col_index.tolist() == rec["colI"] and enc.omega_ptr.tolist() == rec["omegaPtr"]
        assert enc.row_ptr.tolist() == rec["rowPtr"]
        assert [enc.col_index_bits, enc.omega_ptr_bits, enc.row_ptr_bits] == rec["widths"][:3]
        if rec["kind"] == "cser":
            assert enc.omega_index.tolist() == rec["omegaI"] and enc.mode_index == rec["mode_index"]
        assert enc.element_bits == rec["element_bits"]
        cd.write_matrix(out, enc)
        assert open(out, "rb").read() == raw
        # the loaded encoding computes: dot == dense product of its decode
        w = cd.decode(enc).values
        x = np.random.default_rng(0).integers(-3, 4, size=w.shape[1]).astype(np.float64)
        assert np.allclose(cd.dot(enc, x), w @ x, rtol=1e-6, atol=1e-6)


@pytest.mark.gpu
def test_encoder_output_writes_like_reference(lemx_golden, tmp_path):
    """Our GPU encoder + writer reproduce the reference's container bytes for the same matrix."""
    m_rec = [r for r in lemx_golden["files"] if r["matrix"] == 0]
    w = cd.decode(cd.CerMatrix(np.asarray(m_rec[0]["omega"]), np.asarray(m_rec[0]["colI"], np.uint8),
                               np.asarray(m_rec[0]["omegaPtr"], np.uint8), np.asarray(m_rec[0]["rowPtr"], np.uint8),
                               m_rec[0]["m"], m_rec[0]["n"])).values
    path = str(tmp_path / "e.lemx")
    for rec in m_rec:
        enc = (cd.encode_cer if rec["kind"] == "cer" else cd.encode_cser)(cd.DenseMatrix(w, element_bits=rec["element_bits"]))
        cd.write_matrix(path, enc)
        assert open(path, "rb").read() == bytes.fromhex(rec["hex"]), (rec["kind"], rec["element_bits"])
