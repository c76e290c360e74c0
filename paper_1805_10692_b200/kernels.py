"""CER / CSER dot products on the GPU, drop-in for lemt.kernels (kernels.py:53-336).

``dot_cer`` / ``dot_cser`` / ``dot`` call libcerdot's fp32 kernels on the
HBM-resident encoding.  Inputs:

* numpy arrays, ``Vector`` / ``DenseMatrix`` (this package's or the
  reference's) or array-likes -> copied to the device, result returned as a
  float64 numpy array like the reference (computed in fp32);
* CUDA torch tensors -> used in place, result returned as an fp32 CUDA
  tensor on the same stream (no host synchronisation).

``trace=True`` returns ``(y, OpTrace)`` with the reference's analytic
operation counts (kernels.py:175-234), computed on the host from the
encoding's row/segment structure; traces never change numeric results.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .device import require_cuda, stream_ptr, torch_mod
from .formats import (
    TAG_COLI,
    TAG_INPUT,
    TAG_NONE,
    TAG_OMEGA,
    TAG_OMEGAI,
    TAG_OMEGAPTR,
    TAG_OUTPUT,
    TAG_ROWPTR,
    CerMatrix,
    CserMatrix,
)
from .matrices import DenseMatrix, Vector

OP_KINDS = ("sum", "mul", "read", "write", "other")


@dataclass
class OpTrace:
    """Counts of elementary operations keyed by (kind, bits, array tag) (kernels.py:53-95)."""

    counts: dict = field(default_factory=dict)

    def add(self, kind: str, bits: int, tag: str, count: int) -> None:
        if kind not in OP_KINDS:
            raise ValueError(f"unknown op kind {kind!r}")
        if count < 0:
            raise ValueError("counts must be non-negative")
        if count:
            key = (kind, int(bits), tag)
            self.counts[key] = self.counts.get(key, 0) + int(count)

    def merged(self, other: "OpTrace") -> "OpTrace":
        out = OpTrace(dict(self.counts))
        for key, cnt in other.counts.items():
            out.counts[key] = out.counts.get(key, 0) + cnt
        return out

    def scaled(self, factor: int) -> "OpTrace":
        return OpTrace({key: cnt * factor for key, cnt in self.counts.items()})

    def total(self, include_other: bool = False) -> int:
        return sum(c for (k, _, _), c in self.counts.items() if include_other or k != "other")

    def by_kind(self, include_other: bool = False) -> dict:
        out: dict = {}
        for (k, _, _), c in self.counts.items():
            if k == "other" and not include_other:
                continue
            out[k] = out.get(k, 0) + c
        return out

    def count(self, kind: str | None = None, tag: str | None = None) -> int:
        return sum(c for (k, _, t), c in self.counts.items()
                   if (kind is None or k == kind) and (tag is None or t == tag))


# --------------------------------------------------------------------------- host-side input handling


def _input_array(x):
    """(float ndarray, input bits) for host inputs (kernels.py:98-103); fp32/fp64 arrays pass through
    unconverted (the device rounds to fp32 anyway)."""
    if isinstance(x, np.ndarray) and x.dtype in (np.float32, np.float64):
        return x, 32
    if isinstance(x, (Vector, DenseMatrix)) or (hasattr(x, "values") and hasattr(x, "element_bits")):
        return np.asarray(x.values, dtype=np.float64), int(x.element_bits)
    return np.asarray(x, dtype=np.float64), 32


def _check_shape(n: int, shape) -> None:
    if len(shape) not in (1, 2):
        raise ValueError("right-hand side must be a vector or a matrix")
    if shape[0] != n:
        raise ValueError(f"dimension mismatch: matrix has n={n}, input has {shape[0]}")


def _resolve_bits(a, b_in, input_bits, output_bits):
    if input_bits is not None:
        b_in = int(input_bits)
    b_out = max(b_in, a.element_bits) if output_bits is None else int(output_bits)
    return b_in, b_out


# --------------------------------------------------------------------------- analytic traces (kernels.py:175-234)


def _segment_shape(x, rows):
    row_ptr = x.row_ptr.astype(np.int64)
    seg_sizes = np.diff(x.omega_ptr.astype(np.int64))
    segs_per_row = np.diff(row_ptr)
    ne_prefix = np.concatenate(([0], np.cumsum(seg_sizes > 0)))
    sz_prefix = np.concatenate(([0], np.cumsum(seg_sizes)))
    nonempty = ne_prefix[row_ptr[1:]] - ne_prefix[row_ptr[:-1]]
    entries = sz_prefix[row_ptr[1:]] - sz_prefix[row_ptr[:-1]]
    if rows is not None:
        sel = np.asarray(rows)
        return segs_per_row[sel], nonempty[sel], entries[sel]
    return segs_per_row, nonempty, entries


def _device_trace_counts(x):
    """(rows, segments, non-empty, entries, rows with segments, sum max(non-empty - 1, 0)) counted on the
    device (cerdot_trace_counts) for a device-resident encoding, without downloading its arrays."""
    torch = torch_mod()
    dev = x._dev
    ws = torch.zeros(8, dtype=torch.int64, device=dev.device)
    out = (ctypes.c_uint64 * 5)()
    with torch.cuda.device(dev.device):
        _native.check(_native.lib().cerdot_trace_counts(dev.struct(), out, ws.data_ptr(), stream_ptr(dev.device)))
    return (x.m,) + tuple(int(v) for v in out)


def _trace_segmented(x, input_bits, output_bits, rows, columns, with_omega_index) -> OpTrace:
    b_in, b_out = _resolve_bits(x, 32, input_bits, output_bits)
    if rows is None and getattr(x, "_dev", None) is not None:
        r, s, s_ne, z, rows_with_segs, extra_sums = _device_trace_counts(x)
    else:
        segs, nonempty, entries = _segment_shape(x, rows)
        r = len(segs)
        s, s_ne, z = int(segs.sum()), int(nonempty.sum()), int(entries.sum())
        rows_with_segs, extra_sums = int((segs > 0).sum()), int(np.maximum(nonempty - 1, 0).sum())
    t = OpTrace()
    if x.background != 0.0:
        t.add("sum", b_in, TAG_NONE, max(x.n - 1, 0))
        t.add("mul", b_out, TAG_NONE, 1)
        t.add("sum", b_out, TAG_NONE, r + s_ne)
    t.add("read", x.row_ptr_bits, TAG_ROWPTR, 2 * r)
    t.add("read", x.omega_ptr_bits, TAG_OMEGAPTR, s + rows_with_segs)
    if with_omega_index:
        t.add("read", x.omega_index_bits, TAG_OMEGAI, s)
    t.add("read", x.element_bits, TAG_OMEGA, s_ne)
    t.add("read", x.col_index_bits, TAG_COLI, z)
    t.add("read", b_in, TAG_INPUT, z)
    t.add("sum", b_in, TAG_NONE, z - s_ne)
    t.add("mul", b_out, TAG_NONE, s_ne)
    t.add("sum", b_out, TAG_NONE, extra_sums)
    t.add("write", b_out, TAG_OUTPUT, r)
    t.add("other", 0, TAG_NONE, 3 * r + 4 * s + z + 1)
    return t.scaled(columns) if columns != 1 else t


def trace_cer(a: CerMatrix, input_bits: int = 32, output_bits: int | None = None, rows=None,
              columns: int = 1) -> OpTrace:
    return _trace_segmented(a, input_bits, output_bits, rows, columns, with_omega_index=False)


def trace_cser(a: CserMatrix, input_bits: int = 32, output_bits: int | None = None, rows=None,
               columns: int = 1) -> OpTrace:
    return _trace_segmented(a, input_bits, output_bits, rows, columns, with_omega_index=True)


def trace_of(a, input_bits: int = 32, output_bits: int | None = None, rows=None, columns: int = 1) -> OpTrace:
    if isinstance(a, CerMatrix):
        return trace_cer(a, input_bits, output_bits, rows, columns)
    if isinstance(a, CserMatrix):
        return trace_cser(a, input_bits, output_bits, rows, columns)
    raise TypeError(f"not a CER/CSER matrix: {type(a)!r} (dense/CSR are outside this package's scope)")


def row_trace(a, row: int, input_bits: int = 32, output_bits: int | None = None) -> OpTrace:
    """Trace of the scalar product of one matrix row with an input vector (kernels.py:249-251)."""
    return trace_of(a, input_bits, output_bits, rows=[row])


# --------------------------------------------------------------------------- numeric kernels


def _check_out(out, m: int, x, batch: int, keep_2d: bool):
    """Validate a caller-supplied output (kernels write m x batch fp32 through row stride out.stride(0))."""
    torch = torch_mod()
    want = (m, batch) if keep_2d else (m,)
    if not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or out.device != x.device:
        raise ValueError(f"out must be a float32 tensor on {x.device}")
    if tuple(out.shape) != want:
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {want}")
    if out.stride(-1) != 1 or (out.ndim == 2 and batch == 1 and out.stride(0) != 1) or \
            (out.ndim == 2 and out.stride(0) < batch):
        raise ValueError("out must have unit column stride and row stride >= batch")


def dot_device(enc, x, out=None, stream=None, peers=None, peer_offset: int = 0):
    """Device-only entry: ``x`` a CUDA fp32 tensor (n,) or (n, B); returns y (m,) / (m, B) fp32.

    Stream-ordered on ``stream`` (default: torch's current stream of x's device), no host sync.  The
    encoding must live on x's device.  ``out`` (optional) must be float32 on that device with y's shape
    and a unit inner stride.  ``peers``: a CUDA int64 tensor of other ranks' output-buffer addresses;
    every y element is then also stored at element ``peer_offset + i`` of each of them from the kernels'
    epilogue (cerdot_dot_peers, the fused row-sharded all-gather; the caller adds the cross-rank barrier).
    For batch > 1 the dot runs the TMA-staged mat-mat over the encoding's column-tiled view, built on the
    device on the first mat-mat call for that tile height and cached on the encoding.
    """
    torch = torch_mod()
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError("dot_device needs a CUDA tensor input")
    dev = enc._dev if enc._dev is not None else enc.device_encoding(x.device)
    if dev.device != x.device:
        raise ValueError(f"the encoding lives on {dev.device}, the input on {x.device}")
    if x.ndim not in (1, 2) or x.shape[0] != dev.n:
        _check_shape(dev.n, tuple(x.shape))
    if x.dtype != torch.float32:
        x = x.to(torch.float32)
    keep_2d = x.ndim == 2
    batch = int(x.shape[1]) if keep_2d else 1
    if batch == 1:
        if x.ndim == 2:
            x = x.reshape(dev.n)  # an (n, 1) column (a view when its stride allows, else a copy)
        if x.stride(0) != 1:
            x = x.contiguous()
        ldx = 1
    else:
        if x.stride(1) != 1:
            x = x.contiguous()
        ldx = x.stride(0)
    if out is None:
        out = torch.empty((dev.m, batch) if keep_2d else (dev.m,), dtype=torch.float32, device=x.device)
    else:
        _check_out(out, dev.m, x, batch, keep_2d)
    ldy = 1 if (out.ndim == 1 or batch == 1) else out.stride(0)
    with torch.cuda.device(x.device):
        cur = torch.cuda.current_stream(x.device)
        sp = stream if stream is not None else cur.cuda_stream
        st = dev.tile_struct(batch, sp) if batch > 1 else dev.struct()
        # == cerdot_dot_workspace_bytes: the column sums (+ 16 row-range partials each when batch > 1),
        # allocated per call from torch's caching allocator (ordered on the current stream; recorded on a
        # foreign one), so calls on different streams never share scratch
        # (batch > 1: also the tiled mat-mat's tile-split partial products, so the size is asked for)
        if batch > 1:
            ws_bytes = int(_native.lib().cerdot_dot_workspace_bytes(st, batch))
        else:
            ws_bytes = 8 if dev.background != 0.0 else 0
        ws = None
        if ws_bytes:
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=x.device)
            if stream is not None and stream != cur.cuda_stream:
                ws.record_stream(torch.cuda.ExternalStream(stream, device=x.device))
        ws_ptr = ws.data_ptr() if ws is not None else None
        if peers is not None and peers.numel() > 0:
            if peers.dtype != torch.int64 or peers.device != x.device:
                raise ValueError("peers must be an int64 tensor of device pointers on the dot's device")
            _native.check(_native.lib().cerdot_dot_peers(st, x.data_ptr(), ldx, batch, out.data_ptr(), ldy,
                                                          peers.data_ptr(), int(peers.numel()), int(peer_offset),
                                                          ws_ptr, ws_bytes, sp))
            return out
        _native.check(_native.lib().cerdot_dot(st, x.data_ptr(), ldx, batch, out.data_ptr(), ldy, ws_ptr, ws_bytes,
                                               sp))
    return out


class _HostIO(threading.local):
    """Per-thread cached buffers of the host-array path: pinned x / y and the device workspace per shape."""

    def __init__(self):
        self.dev = None
        self.sets = {}
        self.ws_bytes = {}

    def get(self, m: int, n: int, batch: int, ws_bytes: int):
        torch = torch_mod()
        if self.dev is None:
            self.dev = require_cuda()
            self.sets = {}
        key = (m, n, batch)
        bufs = self.sets.get(key)
        if bufs is None or bufs[4].numel() < ws_bytes:
            xs = (n,) if batch == 1 else (n, batch)
            ys = (m,) if batch == 1 else (m, batch)
            px = torch.empty(xs, dtype=torch.float32, pin_memory=True)
            py = torch.empty(ys, dtype=torch.float32, pin_memory=True)
            ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=self.dev)
            bufs = (px, px.numpy(), py, py.numpy(), ws)
            if len(self.sets) > 16:
                self.sets.clear()
            self.sets[key] = bufs
        return bufs


_IO = _HostIO()


def _dot_host(a, xv: np.ndarray) -> np.ndarray:
    """numpy x -> pinned staging -> one C call (cerdot_dot_host: H2D, kernel, D2H, sync) -> float64 numpy
    of the reference's shape ((m,) for a vector, (m, B) for a matrix, including B = 1)."""
    torch = torch_mod()
    batch = 1 if xv.ndim == 1 else int(xv.shape[1])
    if _IO.dev is None:
        _IO.dev = require_cuda()
    dev = a._dev if a._dev is not None else a.device_encoding(_IO.dev)
    if dev.device != _IO.dev:  # run where the encoding lives
        _IO.dev, _IO.sets = dev.device, {}
    st = dev.tile_struct(batch, torch._C._cuda_getCurrentRawStream(_IO.dev.index)) if batch > 1 else dev.struct()
    L = _native.lib()
    key = (a.m, a.n, batch, st.background != 0.0)  # what the workspace size depends on
    ws_bytes = _IO.ws_bytes.get(key)
    if ws_bytes is None:
        ws_bytes = L.cerdot_dot_host_workspace_bytes(st, batch)
        if len(_IO.ws_bytes) > 256:
            _IO.ws_bytes.clear()
        _IO.ws_bytes[key] = ws_bytes
    px, px_np, py, py_np, ws = _IO.get(a.m, a.n, batch, ws_bytes)
    np.copyto(px_np, xv.reshape(px_np.shape), casting="unsafe")  # the kernels compute in fp32
    with torch.cuda.device(_IO.dev):
        _native.check(L.cerdot_dot_host(st, px.data_ptr(), batch, batch, py.data_ptr(), batch, ws.data_ptr(),
                                        ws.numel(), torch._C._cuda_getCurrentRawStream(_IO.dev.index)))
    y = py_np.astype(np.float64)
    return y.reshape(a.m, 1) if (xv.ndim == 2 and batch == 1) else y


class _FastHost(threading.local):
    """Per-thread cache of the e2e host path's fixed call arguments per (encoding, input shape): pinned
    staging views, the device workspace and the prebound C call, so a call is copy-in, one C call
    (H2D, kernel, D2H, sync), copy-out."""

    def __init__(self):
        self.entries = {}


_FAST = _FastHost()
_F_TYPES = (np.float32, np.float64)


def _raw_stream(idx: int) -> int:
    return torch_mod()._C._cuda_getCurrentRawStream(idx)


def _fast_entry(a, shape):
    import weakref

    torch = torch_mod()
    batch = 1 if len(shape) == 1 else int(shape[1])
    if _IO.dev is None:
        _IO.dev = require_cuda()
    dev = a._dev if a._dev is not None else a.device_encoding(_IO.dev)
    if dev.device != _IO.dev:
        _IO.dev, _IO.sets = dev.device, {}
    idx = _IO.dev.index
    st = dev.tile_struct(batch, torch._C._cuda_getCurrentRawStream(idx)) if batch > 1 else dev.struct()
    L = _native.lib()
    ws_bytes = L.cerdot_dot_host_workspace_bytes(st, batch)
    px, px_np, py, py_np, ws = _IO.get(a.m, a.n, batch, ws_bytes)
    call = (L.cerdot_dot_host, (ctypes.byref(st), ctypes.c_void_p(px.data_ptr()), batch, batch,
                                 ctypes.c_void_p(py.data_ptr()), batch, ctypes.c_void_p(ws.data_ptr()), ws.numel()))
    if len(_FAST.entries) > 64:
        _FAST.entries.clear()
    ent = (weakref.ref(a), px_np, py_np, call, idx, (a.m, 1) if len(shape) == 2 and batch == 1 else None,
           (px, py, ws, st))
    _FAST.entries[(id(a), shape)] = ent
    return ent


def _dot_host_fast(a, x: np.ndarray) -> np.ndarray:
    """The e2e host path for numpy float32/float64 inputs: cached arguments (see _FastHost)."""
    ent = _FAST.entries.get((id(a), x.shape))
    if ent is None or ent[0]() is not a:
        ent = _fast_entry(a, x.shape)
    _, px_np, py_np, call, idx, shape2, _keep = ent
    np.copyto(px_np, x.reshape(px_np.shape) if shape2 else x, casting="unsafe")  # the kernels compute in fp32
    rc = call[0](*call[1], _raw_stream(idx))
    if rc:
        _native.check(rc)
    y = py_np.astype(np.float64)
    return y.reshape(shape2) if shape2 else y


def _dot_encoded(a, x, trace, input_bits, output_bits, tracer):
    if not trace and type(x) is np.ndarray and x.dtype.type in _F_TYPES and 1 <= x.ndim <= 2:
        _check_shape(a.n, x.shape)
        return _dot_host_fast(a, x)
    torch = torch_mod()
    if isinstance(x, torch.Tensor):
        _check_shape(a.n, tuple(x.shape))
        if not x.is_cuda:
            x = x.to(require_cuda())
        y = dot_device(a, x)
        b_in = 32
        cols = 1 if x.ndim == 1 else int(x.shape[1])
    else:
        xv, b_in = _input_array(x)
        _check_shape(a.n, xv.shape)
        y = _dot_host(a, xv)
        cols = 1 if xv.ndim == 1 else xv.shape[1]
    if not trace:
        return y
    b_in = b_in if input_bits is None else input_bits
    return y, tracer(a, b_in, output_bits, columns=cols)


def dot_cer(a: CerMatrix, x, trace: bool = False, input_bits: int | None = None, output_bits: int | None = None):
    """y = A.x for a CER matrix (kernels.py:304-312)."""
    if not isinstance(a, CerMatrix):
        raise TypeError(f"dot_cer needs a CerMatrix, got {type(a)!r}")
    return _dot_encoded(a, x, trace, input_bits, output_bits, trace_cer)


def dot_cser(a: CserMatrix, x, trace: bool = False, input_bits: int | None = None, output_bits: int | None = None):
    """y = A.x for a CSER matrix (kernels.py:315-323)."""
    if not isinstance(a, CserMatrix):
        raise TypeError(f"dot_cser needs a CserMatrix, got {type(a)!r}")
    return _dot_encoded(a, x, trace, input_bits, output_bits, trace_cser)


def dot(a, x, trace: bool = False, input_bits: int | None = None, output_bits: int | None = None):
    """Format-dispatched dot product (kernels.py:326-336)."""
    if not trace and type(x) is np.ndarray and (type(a) is CerMatrix or type(a) is CserMatrix) and \
            x.dtype.type in _F_TYPES and 1 <= x.ndim <= 2:
        if x.shape[0] != a.n:
            _check_shape(a.n, x.shape)
        return _dot_host_fast(a, x)
    if isinstance(a, CerMatrix):
        return dot_cer(a, x, trace, input_bits, output_bits)
    if isinstance(a, CserMatrix):
        return dot_cser(a, x, trace, input_bits, output_bits)
    raise TypeError(f"not a matrix: {type(a)!r} (this package implements CER/CSER only)")
