"""LEMX encoded-matrix containers for CER / CSER (lemt io.py:177-278), loaded straight into HBM.

Container layout (little-endian; the reference's io.py docstring)::

    magic b"LEMX" | version u16 | tag u8 (2 cer, 3 cser) | m, n u32 | ebits u8
    cer:  colI, omegaPtr, rowPtr widths u8 | k u32 | nnz, segments u64
    cser: colI, omegaI, omegaPtr, rowPtr widths u8 | mode_index u16 | k u32 | nnz, segments u64
    arrays at their declared widths: omega (element format f64/f32/f16/i8), colI, [omegaI,] omegaPtr, rowPtr

``read_matrix`` parses and checks the header on the host, sends the payload to the device in one copy,
and ``cerdot_lemx_unpack`` scatters it into the encoding's arena (omega widened to f64).  The loaded
encoding is validated on the device (``formats.validate``) before its derived row index is built --
a deviation: the reference's read_matrix does not validate, it fails later in decode.  Dense and CSR
containers are outside this package (IoFormatError "bad-header").  ``write_matrix`` produces
byte-identical containers to the reference's.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _native
from .device import DeviceEncoding, require_cuda, stream_ptr, torch_mod
from .formats import CerMatrix, CserMatrix, validate

MATRIX_MAGIC = b"LEMX"
VERSION = 1
_TAGS = {"dense": 0, "csr": 1, "cer": 2, "cser": 3}
_FIXED = "<HBIIB"
_CER_HDR = "<BBBIQQ"
_CSER_HDR = "<BBBBHIQQ"

__all__ = ["IoFormatError", "read_matrix", "write_matrix", "header_bytes", "MATRIX_MAGIC", "VERSION"]


class IoFormatError(ValueError):
    """File-format failure with a machine-readable code (io.py IoFormatError)."""

    def __init__(self, code: str, message: str):
        self.code = code
        super().__init__(f"{code}: {message}")


def _element_dtype(bits: int) -> np.dtype:
    return {64: np.dtype("<f8"), 32: np.dtype("<f4"), 16: np.dtype("<f2"), 8: np.dtype("<i1")}[bits]


def _index_dtype(bits: int) -> np.dtype:
    return {8: np.dtype("<u1"), 16: np.dtype("<u2"), 32: np.dtype("<u4")}[bits]


def header_bytes(kind: str) -> int:
    """Fixed container header size of a CER / CSER container."""
    return 4 + struct.calcsize(_FIXED) + struct.calcsize(_CER_HDR if kind == "cer" else _CSER_HDR)


def _parse(raw: bytes, path) -> dict:
    if raw[:4] != MATRIX_MAGIC:
        raise IoFormatError("bad-magic", f"not an encoded-matrix container: {path}")
    if len(raw) < 4 + struct.calcsize(_FIXED):
        raise IoFormatError("payload-mismatch", "payload length mismatch reading header")
    version, tag, m, n, ebits = struct.unpack_from(_FIXED, raw, 4)
    if version != VERSION:
        raise IoFormatError("bad-version", f"unsupported version {version}")
    if tag not in (_TAGS["cer"], _TAGS["cser"]):
        raise IoFormatError("bad-header", f"format tag {tag} is not CER/CSER (dense and CSR are out of scope)")
    if ebits not in (8, 16, 32, 64):
        raise IoFormatError("bad-header", f"unsupported element width {ebits}")
    kind = "cer" if tag == _TAGS["cer"] else "cser"
    off = 4 + struct.calcsize(_FIXED)
    fmt = _CER_HDR if kind == "cer" else _CSER_HDR
    if len(raw) < off + struct.calcsize(fmt):
        raise IoFormatError("payload-mismatch", "payload length mismatch reading header")
    fields = struct.unpack_from(fmt, raw, off)
    if kind == "cer":
        cbits, obits, rbits, k, nnz, segs = fields
        widths, mode = {"colI": cbits, "omegaPtr": obits, "rowPtr": rbits}, 0
        order = [("colI", nnz), ("omegaPtr", segs + 1), ("rowPtr", m + 1)]
    else:
        cbits, ibits, obits, rbits, mode, k, nnz, segs = fields
        widths = {"colI": cbits, "omegaI": ibits, "omegaPtr": obits, "rowPtr": rbits}
        order = [("colI", nnz), ("omegaI", segs), ("omegaPtr", segs + 1), ("rowPtr", m + 1)]
    for name, b in widths.items():
        if b not in (8, 16, 32):
            raise IoFormatError("bad-header", f"unsupported {name} width {b}")
    pos = off + struct.calcsize(fmt)
    spans = {"omega": (pos, k * (ebits // 8))}
    pos += k * (ebits // 8)
    for name, count in order:
        spans[name] = (pos, count * widths[name] // 8)
        pos += count * widths[name] // 8
        if pos > len(raw):
            raise IoFormatError("payload-mismatch", f"payload length mismatch reading {name}")
    if spans["omega"][0] + spans["omega"][1] > len(raw):
        raise IoFormatError("payload-mismatch", "payload length mismatch reading values")
    if pos != len(raw):
        raise IoFormatError("payload-mismatch", "payload length mismatch: trailing bytes")
    return {"kind": kind, "m": m, "n": n, "ebits": ebits, "k": k, "nnz": nnz, "segs": segs, "mode": mode,
            "widths": widths, "spans": spans, "payload_at": off + struct.calcsize(fmt)}


def read_matrix(path, device=None):
    """A CER / CSER container as a device-resident encoding (io.py:214-278)."""
    torch = torch_mod()
    dev = require_cuda(device)
    raw = Path(path).read_bytes()
    h = _parse(raw, path)
    kind = _native.CER if h["kind"] == "cer" else _native.CSER
    offsets, total = DeviceEncoding.layout(kind, h["m"], h["k"], h["nnz"], h["segs"], h["widths"])
    base = h["payload_at"]
    staging = torch.frombuffer(bytearray(raw[base:]), dtype=torch.uint8) if len(raw) > base else torch.zeros(
        1, dtype=torch.uint8)
    payload = staging.pin_memory().to(dev, non_blocking=True)
    arena = torch.zeros(total, dtype=torch.uint8, device=dev)
    spans = []
    for name in ("colI", "omegaI", "omegaPtr", "rowPtr"):
        if name in h["widths"]:
            src, nb = h["spans"][name]
            spans += [src - base, offsets[name], nb]
    sp = (np.asarray(spans, dtype=np.int64))
    with torch.cuda.device(dev):
        _native.check(_native.lib().cerdot_lemx_unpack(
            payload.data_ptr(), h["ebits"], h["k"], h["spans"]["omega"][0] - base, arena.data_ptr() + offsets["omega"],
            sp.ctypes.data, len(spans) // 3, arena.data_ptr(), stream_ptr(dev)))
        torch.cuda.current_stream(dev).synchronize()
    omega = np.frombuffer(raw, dtype=_element_dtype(h["ebits"]), count=h["k"],
                          offset=h["spans"]["omega"][0]).astype(np.float64)
    bg = float(omega[h["mode"]] if kind == _native.CSER and h["mode"] < h["k"] else (omega[0] if h["k"] else 0.0))
    checked = DeviceEncoding(kind, h["m"], h["n"], h["k"], h["nnz"], h["segs"], h["mode"], bg, dict(h["widths"]),
                             arena, offsets, 0, 0)
    cls = CerMatrix if kind == _native.CER else CserMatrix
    if kind == _native.CER:
        enc = cls(None, None, None, None, h["m"], h["n"], h["ebits"], _device=checked)
    else:
        enc = cls(None, None, None, None, None, h["m"], h["n"], h["ebits"], h["mode"], _device=checked)
    validate(enc)  # on the device; derived indices only for a structurally valid encoding
    rp = np.frombuffer(raw, dtype=_index_dtype(h["widths"]["rowPtr"]), count=h["m"] + 1,
                       offset=h["spans"]["rowPtr"][0]).astype(np.int64)
    op = np.frombuffer(raw, dtype=_index_dtype(h["widths"]["omegaPtr"]), count=h["segs"] + 1,
                       offset=h["spans"]["omegaPtr"][0]).astype(np.int64)
    checked.max_row_segments = int(np.diff(rp).max()) if h["m"] else 0
    checked.max_row_nnz = int((op[rp[1:]] - op[rp[:-1]]).max()) if h["m"] else 0
    checked._struct = None
    with torch.cuda.device(dev):
        checked.fill_row_entries(stream_ptr(dev))
        torch.cuda.current_stream(dev).synchronize()
    return enc


def write_matrix(path, x) -> None:
    """Write a CER / CSER encoding as a LEMX container (io.py:177-211), byte-identical to lemt's."""
    if not isinstance(x, (CerMatrix, CserMatrix)):
        raise TypeError(f"not a CER/CSER matrix: {type(x)!r}")
    eb = x.element_bits
    omega = np.asarray(x.omega, dtype=np.float64)
    packed = omega.astype(_element_dtype(eb))
    if not np.array_equal(packed.astype(np.float64), omega):
        raise IoFormatError("value-width", f"values are not representable at {eb} bits")
    out = bytearray(MATRIX_MAGIC)
    cer = isinstance(x, CerMatrix)
    out += struct.pack(_FIXED, VERSION, _TAGS["cer" if cer else "cser"], x.m, x.n, eb)
    if cer:
        out += struct.pack(_CER_HDR, x.col_index_bits, x.omega_ptr_bits, x.row_ptr_bits, omega.size, x.nnz,
                           x.segment_count)
        arrays = [(x.col_index, x.col_index_bits), (x.omega_ptr, x.omega_ptr_bits), (x.row_ptr, x.row_ptr_bits)]
    else:
        out += struct.pack(_CSER_HDR, x.col_index_bits, x.omega_index_bits, x.omega_ptr_bits, x.row_ptr_bits,
                           x.mode_index, omega.size, x.nnz, x.segment_count)
        arrays = [(x.col_index, x.col_index_bits), (x.omega_index, x.omega_index_bits),
                  (x.omega_ptr, x.omega_ptr_bits), (x.row_ptr, x.row_ptr_bits)]
    out += packed.tobytes()
    for arr, bits in arrays:
        out += np.asarray(arr).astype(_index_dtype(bits)).tobytes()
    Path(path).write_bytes(bytes(out))
