"""Device residency of CER/CSER encodings.

HBM layout of one encoding: a single ``uint8`` arena (one allocation, one
H2D/D2H copy when it crosses the bus) holding, each 256-byte aligned,

    omega        k   float64   (CER frequency-major / CSER value-ascending)
    colI         nnz uint{8,16,32}
    omegaPtr     S+1 uint{8,16,32}
    rowPtr       m+1 uint{8,16,32}
    omegaI       S   uint{8,16,32}   (CSER only)
    rowEntry     m+1 uint32          (derived index: omegaPtr[rowPtr[r]], see
                                      cerdot_row_entries; not part of the format)

at exactly the reference's per-array widths, so the bytes the dot kernels
stream are the reference's ``storage_bits`` (plus omega at 8 B instead of
the 4 B ``element_bits`` accounting).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _native

_NP_UINT = {8: np.uint8, 16: np.uint16, 32: np.uint32}
_ALIGN = 256


def torch_mod():
    import torch  # plumbing only: device memory and streams

    return torch


def require_cuda(device=None):
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1805_10692_b200 runs on a CUDA (sm_100a) device and has no CPU fallback; "
            "torch.cuda.is_available() is False")
    _native.lib()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"expected a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_ptr(device=None) -> int:
    torch = torch_mod()
    return torch.cuda.current_stream(device).cuda_stream


def ctypes_copy(dst, src) -> None:
    import ctypes

    ctypes.memmove(ctypes.addressof(dst), ctypes.addressof(src), ctypes.sizeof(src))


def _align(v: int) -> int:
    return (v + _ALIGN - 1) // _ALIGN * _ALIGN


@dataclass
class DeviceEncoding:
    kind: int  # _native.CER / CSER
    m: int
    n: int
    k: int
    nnz: int
    segments: int
    mode_index: int
    background: float
    bits: dict  # name -> 8/16/32 for colI, omegaPtr, rowPtr, omegaI
    arena: object  # torch.uint8 cuda tensor
    offsets: dict  # name -> byte offset
    max_row_nnz: int = 0  # largest row in entries (0 = unknown)
    max_row_segments: int = 0  # largest row in segments (0 = unknown)
    _struct: object = field(default=None, repr=False)
    _row_entry_ready: bool = False
    _tile_views: dict = field(default_factory=dict, repr=False)  # NT -> (tile_ptr, tile_rec, struct)

    def fill_row_entries(self, stream: int) -> None:
        """Compute the derived rowEntry index on the device (stream-ordered)."""
        if "rowEntry" not in self.offsets:
            return
        self._row_entry_ready = False
        self._struct = None
        _native.check(_native.lib().cerdot_row_entries(self.struct(), self.ptr("rowEntry"), stream))
        self._row_entry_ready = True
        self._struct = None

    def tile_struct(self, batch: int, stream: int):
        """The matrix struct carrying the column-tiled view the mat-mat wants at this batch (built on the
        device on first use, stream-ordered, then cached), or the plain struct when no view applies."""
        base = self.struct()
        if batch <= 1 or base.row_entry is None:
            return base
        L = _native.lib()
        nt = int(L.cerdot_tile_view_rows(base, batch))
        if nt <= 0:
            return base
        hit = self._tile_views.get(nt)
        if hit is None:
            torch = torch_mod()
            if torch.cuda.is_current_stream_capturing():
                # building the view inside a user's CUDA-graph capture would make every replay rebuild it:
                # use the flat kernel for this call (run one batched call before capturing to get the view)
                return base
            tiles = -(-self.n // nt)
            tptr = torch.empty(tiles * self.m + 1, dtype=torch.int32, device=self.device)
            rec = torch.empty(max(1, self.nnz) * 2, dtype=torch.int32, device=self.device)
            ws = torch.empty(max(256, int(L.cerdot_tile_view_workspace_bytes(base, nt))), dtype=torch.uint8,
                             device=self.device)
            _native.check(L.cerdot_tile_view_build(base, nt, tptr.data_ptr(), rec.data_ptr(), ws.data_ptr(),
                                                   ws.numel(), stream))
            s = _native.CerdotMatrix()
            ctypes_copy(s, base)
            s.tile_rows, s.tile_ptr, s.tile_rec = nt, tptr.data_ptr(), rec.data_ptr()
            hit = (tptr, rec, s, ws)  # ws kept alive until the build has run (stream-ordered)
            self._tile_views[nt] = hit
        return hit[2]

    @property
    def tile_view_bytes(self) -> int:
        """Device bytes held by the cached column-tiled views (derived indices)."""
        return sum(v[0].numel() * 4 + v[1].numel() * 4 for v in self._tile_views.values())

    @staticmethod
    def layout(kind: int, m: int, k: int, nnz: int, segments: int, bits: dict):
        names = [("omega", k, 64), ("colI", nnz, bits["colI"]), ("omegaPtr", segments + 1, bits["omegaPtr"]),
                 ("rowPtr", m + 1, bits["rowPtr"])]
        if kind == _native.CSER:
            names.append(("omegaI", segments, bits["omegaI"]))
        if nnz < 2**32:
            names.append(("rowEntry", m + 1, 32))
        offsets, off = {}, 0
        for name, count, b in names:
            offsets[name] = off
            off = _align(off + count * (b // 8))
        return offsets, max(off, _ALIGN)

    def count(self, name: str) -> int:
        return {"omega": self.k, "colI": self.nnz, "omegaPtr": self.segments + 1, "rowPtr": self.m + 1,
                "omegaI": self.segments, "rowEntry": self.m + 1}[name]

    def ptr(self, name: str) -> int:
        return self.arena.data_ptr() + self.offsets[name]

    def nbytes(self, name: str) -> int:
        b = 64 if name == "omega" else (32 if name == "rowEntry" else self.bits[name])
        return self.count(name) * (b // 8)

    def to_host(self, name: str) -> np.ndarray:
        start = self.offsets[name]
        raw = self.arena[start:start + self.nbytes(name)].cpu().numpy()
        dt = np.float64 if name == "omega" else (np.uint32 if name == "rowEntry" else _NP_UINT[self.bits[name]])
        arr = raw.view(dt).copy()
        arr.setflags(write=False)
        return arr

    def struct(self) -> "_native.CerdotMatrix":
        if self._struct is None:
            s = _native.CerdotMatrix()
            s.kind = self.kind
            s.mode_index = self.mode_index
            s.m, s.n, s.k, s.nnz, s.segments = self.m, self.n, self.k, self.nnz, self.segments
            s.omega = self.ptr("omega")
            s.col_index = self.ptr("colI")
            s.omega_ptr = self.ptr("omegaPtr")
            s.row_ptr = self.ptr("rowPtr")
            s.omega_index = self.ptr("omegaI") if self.kind == _native.CSER else None
            s.col_bits = self.bits["colI"]
            s.omega_ptr_bits = self.bits["omegaPtr"]
            s.row_ptr_bits = self.bits["rowPtr"]
            s.omega_index_bits = self.bits.get("omegaI", 8)
            s.background = self.background
            s.max_row_nnz = self.max_row_nnz
            s.max_row_segments = self.max_row_segments
            use_re = self._row_entry_ready and not os.environ.get("CERDOT_NO_ROW_ENTRY")
            s.row_entry = self.ptr("rowEntry") if use_re else None
            self._struct = s
        return self._struct

    @property
    def device(self):
        return self.arena.device

    @property
    def format_bytes(self) -> int:
        """Bytes of the encoding's format arrays (the derived rowEntry index excluded)."""
        return sum(self.nbytes(nm) for nm in self.offsets if nm != "rowEntry")

    @classmethod
    def from_host(cls, kind: int, m: int, n: int, mode_index: int, arrays: dict, device=None,
                  derive: bool = True) -> "DeviceEncoding":
        """Upload host arrays (any unsigned-representable ints) narrowed to 8/16/32 bits.  ``derive=False``
        skips the row statistics and the rowEntry index, which index through the pointers: the upload
        of an untrusted encoding for validation."""
        torch = torch_mod()
        dev = require_cuda(device)
        omega = np.ascontiguousarray(arrays["omega"], dtype=np.float64)
        bits, host = {}, {}
        for name in ("colI", "omegaPtr", "rowPtr", "omegaI"):
            if name not in arrays:
                continue
            a = np.asarray(arrays[name])
            mx = int(a.max()) if a.size else 0
            if a.size and int(a.min()) < 0:
                raise ValueError(f"{name}: index values are unsigned")
            b = a.dtype.itemsize * 8 if a.dtype.kind == "u" and a.dtype.itemsize <= 4 else None
            if b is None or (mx >> b):
                b = _native.lib().cerdot_index_bitwidth(mx)
                if b == 0:
                    raise ValueError(_native.last_error())
            bits[name] = b
            host[name] = np.ascontiguousarray(a, dtype=_NP_UINT[b])
        k, nnz, segs = omega.size, host["colI"].size, host["omegaPtr"].size - 1
        offsets, total = cls.layout(kind, m, k, nnz, segs, bits)
        staging = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        buf = staging.numpy()
        buf[offsets["omega"]:offsets["omega"] + omega.nbytes] = omega.view(np.uint8)
        for name, a in host.items():
            buf[offsets[name]:offsets[name] + a.nbytes] = a.view(np.uint8)
        arena = staging.to(dev, non_blocking=True)
        bi = mode_index if kind == _native.CSER else 0
        bg = float(omega[bi]) if 0 <= bi < k else 0.0  # (an out-of-range mode_index is validate's to report)
        if not derive:
            enc = cls(kind, m, n, k, nnz, segs, mode_index, bg, bits, arena, offsets, 0, 0)
            torch.cuda.current_stream(dev).synchronize()  # the pinned staging buffer goes out of scope
            return enc
        rp = host["rowPtr"].astype(np.int64)
        optr = host["omegaPtr"].astype(np.int64)
        seg_rows = np.diff(rp) if m else np.zeros(0, dtype=np.int64)
        nnz_rows = (optr[rp[1:]] - optr[rp[:-1]]) if m else np.zeros(0, dtype=np.int64)
        enc = cls(kind, m, n, k, nnz, segs, mode_index, bg, bits, arena, offsets,
                  int(nnz_rows.max()) if nnz_rows.size else 0, int(seg_rows.max()) if seg_rows.size else 0)
        with torch.cuda.device(dev):
            enc.fill_row_entries(stream_ptr(dev))
            torch.cuda.current_stream(dev).synchronize()
        return enc

