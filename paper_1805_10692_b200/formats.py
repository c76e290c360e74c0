"""CER / CSER encodings, drop-in for lemt.formats (formats.py:42-295, 427-503).

``encode_cer`` / ``encode_cser`` run the conversion on the GPU
(libcerdot: cerdot_encode_plan + cerdot_encode_fill) and return encodings
whose arrays stay resident in HBM.  The reference's field names and
properties (``omega``, ``col_index``, ``omega_ptr``, ``row_ptr``,
``omega_index``, ``mode_index``, ``nnz``, ``segment_count``, ``*_bits``)
are preserved; the numpy views are fetched lazily (one D2H copy per array,
cached) so reference-style code such as ``enc.col_index.tolist()`` keeps
working.  Constructing an encoding from host arrays (as the reference's
tests do to build corrupted copies) is also supported; such an encoding is
uploaded on its first dot product.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .device import DeviceEncoding, require_cuda, stream_ptr, torch_mod
from .matrices import DenseMatrix

INDEX_BITS = (8, 16, 32)

# Array tags used by traces (formats.py:31-39).
TAG_INPUT = "input"
TAG_OUTPUT = "output"
TAG_OMEGA = "omega"
TAG_COLI = "colI"
TAG_OMEGAI = "omegaI"
TAG_OMEGAPTR = "omegaPtr"
TAG_ROWPTR = "rowPtr"
TAG_NONE = "none"


class FormatError(ValueError):
    """Structural validation failure, naming the offending array and offset (formats.py:42-49)."""

    def __init__(self, array: str, offset: int, reason: str):
        self.array = array
        self.offset = offset
        self.reason = reason
        super().__init__(f"{array}[{offset}]: {reason}")


def index_bitwidth(max_index_value: int) -> int:
    """Smallest of 8/16/32 bits that holds the value unsigned (formats.py:52-59; cerdot_index_bitwidth)."""
    bits = _native.lib().cerdot_index_bitwidth(int(max_index_value))
    if bits == 0:
        raise ValueError(_native.last_error())
    return bits


def _resolve_bits(max_value: int, index_bits) -> int:
    """Width for one array with the reference's checks and messages (formats.py:66-71)."""
    bits = index_bitwidth(max_value) if index_bits == "auto" else int(index_bits)
    if bits not in INDEX_BITS:
        raise ValueError(f"index bits must be one of {INDEX_BITS}")
    if max_value >= (1 << bits):
        raise ValueError(f"index value {max_value} does not fit in {bits} bits")
    return bits


_HOST_NAMES = {"omega": "omega", "col_index": "colI", "omega_ptr": "omegaPtr", "row_ptr": "rowPtr",
               "omega_index": "omegaI"}


class _Encoded:
    """Shared machinery: lazy host views over a device-resident encoding."""

    _kind = None
    _fields = ()

    def _setup(self, arrays: dict, m: int, n: int, element_bits: int, mode_index: int, dev: DeviceEncoding | None):
        object.__setattr__(self, "_host", {})
        object.__setattr__(self, "_dev", dev)
        object.__setattr__(self, "m", int(m))
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "element_bits", int(element_bits))
        object.__setattr__(self, "mode_index", int(mode_index))
        for name, arr in arrays.items():
            if arr is None:
                continue
            if hasattr(arr, "detach"):  # torch tensor given directly
                arr = arr.detach().cpu().numpy()
            a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64) if name == "omega" else np.asarray(arr))
            a.setflags(write=False)
            self._host[name] = a

    def __setattr__(self, key, value):
        raise AttributeError(f"cannot assign to field {key!r}: encodings are immutable")

    def _array(self, name: str) -> np.ndarray:
        arr = self._host.get(name)
        if arr is None:
            arr = self._dev.to_host(_HOST_NAMES[name])
            self._host[name] = arr
        return arr

    # ---- reference fields (formats.py:105-170)
    @property
    def omega(self) -> np.ndarray:
        return self._array("omega")

    @property
    def col_index(self) -> np.ndarray:
        return self._array("col_index")

    @property
    def omega_ptr(self) -> np.ndarray:
        return self._array("omega_ptr")

    @property
    def row_ptr(self) -> np.ndarray:
        return self._array("row_ptr")

    def _bits(self, name: str) -> int:
        if name not in self._host and self._dev is not None:
            return self._dev.bits[_HOST_NAMES[name]]
        return self._array(name).dtype.itemsize * 8

    @property
    def nnz(self) -> int:
        return self._dev.nnz if "col_index" not in self._host and self._dev is not None else len(self.col_index)

    @property
    def segment_count(self) -> int:
        if "omega_ptr" not in self._host and self._dev is not None:
            return self._dev.segments
        return len(self.omega_ptr) - 1

    @property
    def col_index_bits(self) -> int:
        return self._bits("col_index")

    @property
    def omega_ptr_bits(self) -> int:
        return self._bits("omega_ptr")

    @property
    def row_ptr_bits(self) -> int:
        return self._bits("row_ptr")

    # ---- device side
    def device_encoding(self, device=None) -> DeviceEncoding:
        """The HBM-resident encoding (uploaded from the host arrays on first use).

        Host-constructed arrays are untrusted: they are validated on the device first (``validate``,
        FormatError on a violation), because the kernels index x and shared memory with colI / omegaI
        unchecked and an out-of-range index would fault the whole CUDA context (the reference raises
        IndexError).  Encodings made by encode_* / read_matrix / the device slicer are device-resident from
        the start and never take this path."""
        if self._dev is None:
            validate(self)
            arrays = {"omega": self.omega, "colI": self.col_index, "omegaPtr": self.omega_ptr,
                      "rowPtr": self.row_ptr}
            if self._kind == _native.CSER:
                arrays["omegaI"] = self.omega_index
            object.__setattr__(self, "_dev", DeviceEncoding.from_host(self._kind, self.m, self.n, self.mode_index,
                                                                       arrays, device))
        return self._dev

    @property
    def background(self) -> float:
        if self._dev is not None:
            return self._dev.background
        om = self.omega
        return float(om[self.mode_index] if self._kind == _native.CSER else om[0])

    def __repr__(self):
        where = "device" if self._dev is not None else "host"
        return (f"{type(self).__name__}(m={self.m}, n={self.n}, k={len(self.omega)}, nnz={self.nnz}, "
                f"segments={self.segment_count}, {where})")


class CerMatrix(_Encoded):
    """Compressed Entropy Row matrix (formats.py:105-133).

    Fields: omega (frequency-major alphabet, omega[0] the background),
    col_index, omega_ptr (segment boundaries, leading 0), row_ptr (m+1
    boundaries into the segment list), m, n, element_bits.
    """

    _kind = _native.CER

    def __init__(self, omega, col_index, omega_ptr, row_ptr, m, n, element_bits=32, *, _device=None):
        self._setup({"omega": omega, "col_index": col_index, "omega_ptr": omega_ptr, "row_ptr": row_ptr},
                    m, n, element_bits, 0, _device)


class CserMatrix(_Encoded):
    """Compressed Shared Elements Row matrix (formats.py:136-170).

    Fields: omega (value-ascending alphabet), col_index, omega_index
    (per-segment position in omega), omega_ptr, row_ptr, m, n,
    element_bits, mode_index (position of the background in omega).
    """

    _kind = _native.CSER

    def __init__(self, omega, col_index, omega_index, omega_ptr, row_ptr, m, n, element_bits=32, mode_index=0, *,
                 _device=None):
        self._setup({"omega": omega, "col_index": col_index, "omega_index": omega_index, "omega_ptr": omega_ptr,
                     "row_ptr": row_ptr}, m, n, element_bits, mode_index, _device)

    @property
    def omega_index(self) -> np.ndarray:
        return self._array("omega_index")

    @property
    def omega_index_bits(self) -> int:
        return self._bits("omega_index")


EncodedMatrix = CerMatrix | CserMatrix


# --------------------------------------------------------------------------- validate / decode

# cerdot_check id -> (array, reason template); {v} is the record's value, {last}/{n}/{k1} the sizes
_CHECKS = {
    1: ("omegaPtr", "must start at 0, found {v}"),
    2: ("omegaPtr", "must be non-decreasing"),
    3: ("omegaPtr", "must end at {nnz}, found {v}"),
    4: ("rowPtr", "must start at 0, found {v}"),
    5: ("rowPtr", "must be non-decreasing"),
    6: ("rowPtr", "must end at {segs}, found {v}"),
    7: ("colI", "column {v} out of range for n={n}"),
    8: ("colI", "must be strictly ascending within a segment"),
    9: ("colI", "duplicate column within a row"),
    10: ("rowPtr", "row holds {v} segments, alphabet has {k1} non-background elements"),
    11: ("omegaPtr", "trailing empty segment"),
    12: ("omegaI", "element index out of range"),
    13: ("omegaI", "segment references the background element"),
    14: ("omegaPtr", "empty segment"),
    15: ("omegaI", "row references an element twice"),
}
_LAST_COLUMN_CHECK = 9


def _device_checks(x, device=None):
    """Run cerdot_validate on the encoding (a validation-only upload of host-constructed arrays: no
    derived indices).  Returns the error record's (check, offset, value)."""
    torch = torch_mod()
    dev = x._dev
    if dev is None:
        arrays = {"omega": x.omega, "colI": x.col_index, "omegaPtr": x.omega_ptr, "rowPtr": x.row_ptr}
        if x._kind == _native.CSER:  # length errors are reported later, in the reference's order
            segs = len(x.omega_ptr) - 1
            oi = np.asarray(x.omega_index)
            arrays["omegaI"] = oi[:segs] if oi.size >= segs else np.concatenate(
                [oi, np.zeros(segs - oi.size, dtype=oi.dtype)])
        dev = DeviceEncoding.from_host(x._kind, x.m, x.n, x.mode_index, arrays, device, derive=False)
    L = _native.lib()
    st = dev.struct()
    nbytes = L.cerdot_validate_workspace_bytes(st)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev.device)
    rec = _native.CerdotFormatError()
    with torch.cuda.device(dev.device):
        rc = L.cerdot_validate(st, ctypes.byref(rec), ws.data_ptr(), nbytes, stream_ptr(dev.device))
    if rc not in (_native.OK, _native.E_FORMAT):
        _native.check(rc)
    return rec.check, rec.offset, rec.value


def validate(x) -> None:
    """Raise FormatError on any structural inconsistency (formats.py:331-392), checked on the device.

    The alphabet and length checks run here (host, tiny arrays); the index arrays are checked by
    ``cerdot_validate`` in the reference's order, so the same first violation is reported.
    """
    if not isinstance(x, (CerMatrix, CserMatrix)):
        raise TypeError(f"not an encoded matrix: {type(x)!r}")
    omega = np.asarray(x.omega, dtype=np.float64)
    k = omega.size
    if np.unique(omega).size != k:
        raise FormatError("omega", 0, "duplicate alphabet values")
    if len(x.row_ptr) != x.m + 1:
        raise FormatError("rowPtr", 0, f"expected {x.m + 1} entries")
    if len(x.omega_ptr) == 0:
        raise FormatError("omegaPtr", 0, "array is empty")
    check, offset, value = _device_checks(x)
    sizes = {"nnz": x.nnz, "segs": len(x.omega_ptr) - 1, "n": x.n, "k1": k - 1}

    def fail(c):
        array, reason = _CHECKS[c]
        raise FormatError(array, int(offset), reason.format(v=int(value), **sizes))

    if check and (check <= _LAST_COLUMN_CHECK or isinstance(x, CerMatrix)):
        fail(check)
    if isinstance(x, CserMatrix):
        if np.any(np.diff(omega) <= 0):
            raise FormatError("omega", 0, "alphabet must be value-ascending")
        segs = len(x.omega_ptr) - 1
        if len(x.omega_index) != segs:
            raise FormatError("omegaI", 0, f"expected {segs} entries, found {len(x.omega_index)}")
        if not 0 <= x.mode_index < k:
            raise FormatError("omega", x.mode_index, "mode_index out of range")
        if check:
            fail(check)


def decode(x):
    """Exact dense reconstruction (formats.py:395-424) on the device; validates first."""
    if isinstance(x, DenseMatrix):
        return x
    validate(x)
    torch = torch_mod()
    dev = x.device_encoding()
    out = torch.empty((x.m, x.n), dtype=torch.float64, device=dev.device)
    with torch.cuda.device(dev.device):
        _native.check(_native.lib().cerdot_decode(dev.struct(), out.data_ptr(), max(x.n, 1), stream_ptr(dev.device)))
    return DenseMatrix(out.cpu().numpy(), element_bits=x.element_bits)


# --------------------------------------------------------------------------- conversion


def _dense_source(a):
    """(device tensor f32/f64 contiguous, element_bits) for any supported dense input."""
    torch = torch_mod()
    if isinstance(a, torch.Tensor):
        if a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got shape {tuple(a.shape)}")
        dev = require_cuda(a.device if a.is_cuda else None)
        if a.dtype not in (torch.float32, torch.float64):
            a = a.to(torch.float64)
        return a.to(dev).contiguous(), 32
    values = getattr(a, "values", a)
    bits = int(getattr(a, "element_bits", 32))
    arr = np.asarray(values)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-d array, got shape {arr.shape}")
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    dev = require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.numel():
        t = t.pin_memory().to(dev, non_blocking=True)
    else:
        t = t.to(dev)
    return t, bits


def _plan(a, background):
    """Shared first half of a conversion: alphabet, ranks, row statistics (one host synchronisation).
    Returns what either format's fill needs; the workspace holds the rank grid until both are done."""
    torch = torch_mod()
    w, element_bits = _dense_source(a)
    m, n = int(w.shape[0]), int(w.shape[1])
    L = _native.lib()
    info = _native.CerdotEncodeInfo()
    ws_bytes = L.cerdot_encode_workspace_bytes(m, n)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=w.device)
    dtype = _native.F32 if w.dtype == torch.float32 else _native.F64
    bg_mode = 0 if background is None else 1
    bg_value = 0.0 if background is None else float(background)
    with torch.cuda.device(w.device):
        st = stream_ptr(w.device)
        rc = L.cerdot_encode_plan(w.data_ptr() if w.numel() else None, dtype, m, n, n, bg_mode, bg_value,
                                  ws.data_ptr(), ws_bytes, info, st)
        if rc == _native.E_WORKSPACE and info.workspace_bytes > ws_bytes:
            # large alphabet: the sort-based conversion needs more scratch; plan again with it
            ws_bytes = info.workspace_bytes
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device=w.device)
            rc = L.cerdot_encode_plan(w.data_ptr(), dtype, m, n, n, bg_mode, bg_value, ws.data_ptr(), ws_bytes, info,
                                      st)
        _native.check(rc)
    return w, element_bits, info, ws, ws_bytes


def _fill(plan, kind: int, index_bits):
    """Second half: allocate the encoding at the planned sizes and write its arrays."""
    torch = torch_mod()
    w, element_bits, info, ws, ws_bytes = plan
    m, n = int(w.shape[0]), int(w.shape[1])
    L = _native.lib()
    with torch.cuda.device(w.device):
        st = stream_ptr(w.device)
        segs = info.segments_cser if kind == _native.CSER else info.segments_cer
        bits = {"colI": _resolve_bits(max(n - 1, 0), index_bits)}
        if kind == _native.CSER:
            bits["omegaI"] = _resolve_bits(max(info.k - 1, 0), index_bits)
        bits["omegaPtr"] = _resolve_bits(max(info.nnz, 0), index_bits)
        bits["rowPtr"] = _resolve_bits(max(segs, 0), index_bits)
        offsets, total = DeviceEncoding.layout(kind, m, info.k, info.nnz, segs, bits)
        arena = torch.empty(total, dtype=torch.uint8, device=w.device)
        dev = DeviceEncoding(kind, m, n, info.k, info.nnz, segs, info.mode_index if kind == _native.CSER else 0,
                             0.0, bits, arena, offsets, int(info.max_row_nnz),
                             int(info.max_row_segments_cser if kind == _native.CSER else info.max_row_segments_cer))
        _native.check(L.cerdot_encode_fill(info, kind, ws.data_ptr(), ws_bytes, dev.ptr("omega"), dev.ptr("colI"),
                                           bits["colI"], dev.ptr("omegaPtr"), bits["omegaPtr"], dev.ptr("rowPtr"),
                                           bits["rowPtr"], dev.ptr("omegaI") if kind == _native.CSER else None,
                                           bits.get("omegaI", 8), st))
        dev.fill_row_entries(st)
    # background as stored in omega (CER omega[0]; CSER omega[mode_index]) — same value
    dev.background = float(info.background)
    dev._struct = None
    if kind == _native.CSER:
        return CserMatrix(None, None, None, None, None, m, n, element_bits, dev.mode_index, _device=dev)
    return CerMatrix(None, None, None, None, m, n, element_bits, _device=dev)


def _encode(a, kind: int, index_bits, background):
    return _fill(_plan(a, background), kind, index_bits)  # the workspace is released stream-ordered


def encode_pair(a, index_bits="auto", background=None):
    """(CerMatrix, CserMatrix) of the same matrix from ONE plan: the alphabet, the rank grid and the row
    statistics are shared (formats.py:193-224 run once), only the two fills differ.  Equal, array by
    array, to encode_cer(a) and encode_cser(a); an extension over the reference's API."""
    plan = _plan(a, background)
    return _fill(plan, _native.CER, index_bits), _fill(plan, _native.CSER, index_bits)


def encode_cer(a, index_bits="auto", background=None) -> CerMatrix:
    """Compressed entropy row encoding on the GPU (formats.py:227-256).

    ``background`` designates the element whose positions are never stored;
    it defaults to the matrix mode (ties broken by ascending value).  A
    background absent from the matrix is allowed and heads the alphabet.
    ``a`` may be a DenseMatrix (this package's or the reference's), a 2-d
    numpy array, or a 2-d torch tensor (CUDA tensors are encoded in place).
    """
    return _encode(a, _native.CER, index_bits, background)


def encode_cser(a, index_bits="auto", background=None) -> CserMatrix:
    """Compressed shared-elements row encoding on the GPU (formats.py:259-295)."""
    return _encode(a, _native.CSER, index_bits, background)


# --------------------------------------------------------------------------- counters (host, formats.py:427-503)


def entry_count(x) -> dict[str, int]:
    """Number of stored entries per array plus their total (formats.py:427-451)."""
    if isinstance(x, DenseMatrix) or (hasattr(x, "values") and hasattr(x, "element_bits") and not
                                      isinstance(x, _Encoded)):
        counts = {"values": int(np.asarray(x.values).size)}
    elif isinstance(x, CerMatrix):
        counts = {"omega": len(x.omega), "colI": x.nnz, "omegaPtr": x.segment_count + 1, "rowPtr": x.m + 1}
    elif isinstance(x, CserMatrix):
        counts = {"omega": len(x.omega), "colI": x.nnz, "omegaI": x.segment_count,
                  "omegaPtr": x.segment_count + 1, "rowPtr": x.m + 1}
    else:
        raise TypeError(f"not a matrix: {type(x)!r}")
    counts["total"] = sum(counts.values())
    return counts


def storage_bits(x) -> int:
    """Exact payload size: sum over arrays of length x bit-width (formats.py:454-479)."""
    if isinstance(x, _Encoded):
        bits = (len(x.omega) * x.element_bits + x.nnz * x.col_index_bits
                + (x.segment_count + 1) * x.omega_ptr_bits + (x.m + 1) * x.row_ptr_bits)
        if isinstance(x, CserMatrix):
            bits += x.segment_count * x.omega_index_bits
        return bits
    if hasattr(x, "values") and hasattr(x, "element_bits"):
        return int(np.asarray(x.values).size) * int(x.element_bits)
    raise TypeError(f"not a matrix: {type(x)!r}")


def array_bytes(x, input_bits: int = 32, output_bits: int | None = None) -> dict[str, float]:
    """Byte size of every addressable array (formats.py:482-503)."""
    if output_bits is None:
        output_bits = max(input_bits, x.element_bits)
    sizes = {TAG_INPUT: x.n * input_bits / 8, TAG_OUTPUT: x.m * output_bits / 8}
    if isinstance(x, _Encoded):
        sizes[TAG_OMEGA] = len(x.omega) * x.element_bits / 8
        sizes[TAG_COLI] = x.nnz * x.col_index_bits / 8
        sizes[TAG_OMEGAPTR] = (x.segment_count + 1) * x.omega_ptr_bits / 8
        sizes[TAG_ROWPTR] = (x.m + 1) * x.row_ptr_bits / 8
        if isinstance(x, CserMatrix):
            sizes[TAG_OMEGAI] = x.segment_count * x.omega_index_bits / 8
    else:
        sizes[TAG_OMEGA] = int(np.asarray(x.values).size) * x.element_bits / 8
    return sizes
