"""TEST INFRASTRUCTURE ONLY — ctypes wrapper for ``cer_oracle.c``.

Same return shapes as :mod:`oracle.numpy_port` (dicts of numpy arrays with
the reference's auto/forced widths).  Builds ``oracle/_build`` on demand
with ``make`` when the library is missing (the GPU box receives the prebuilt
``.so`` with the repo snapshot).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import numpy_port

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcer_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "cer_oracle.c")
        ):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_encode_begin.restype = ctypes.c_void_p
        L.oracle_encode_begin.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_int)]
        L.oracle_encode_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_encode_fill.restype = ctypes.c_int64
        L.oracle_encode_fill.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 5
        L.oracle_encode_free.argtypes = [ctypes.c_void_p]
        L.oracle_dot.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 4 + [ctypes.c_double,
                                                                                  ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def encode(values: np.ndarray, kind: str, index_bits="auto", background=None) -> dict:
    w = np.ascontiguousarray(values)
    if w.dtype not in (np.float32, np.float64):
        w = w.astype(np.float64)
    if w.ndim != 2:
        raise ValueError(f"expected a 2-d array, got shape {w.shape}")
    m, n = w.shape
    err = ctypes.c_int(0)
    h = lib().oracle_encode_begin(_ptr(w), int(w.dtype == np.float32), m, n, int(background is not None),
                                  float(background) if background is not None else 0.0, ctypes.byref(err))
    if err.value == 1:
        raise IndexError("index 0 is out of bounds for axis 0 with size 0")
    if not h:
        raise MemoryError("oracle encode allocation failed")
    try:
        sizes = np.zeros(4, dtype=np.int64)
        lib().oracle_encode_sizes(h, _ptr(sizes))
        k, nnz, s_cer, s_cser = (int(v) for v in sizes)
        s = s_cer if kind == "cer" else s_cser
        omega = np.empty(k, dtype=np.float64)
        col = np.empty(nnz, dtype=np.int64)
        optr = np.empty(s + 1, dtype=np.int64)
        rptr = np.empty(m + 1, dtype=np.int64)
        oidx = np.empty(max(s, 1), dtype=np.int64)
        mode = lib().oracle_encode_fill(h, 0 if kind == "cer" else 1, _ptr(omega), _ptr(col), _ptr(optr),
                                        _ptr(rptr), _ptr(oidx))
    finally:
        lib().oracle_encode_free(h)
    out = {
        "kind": kind, "m": m, "n": n, "omega": omega,
        "colI": numpy_port.as_index(col, max(n - 1, 0), index_bits),
        "omegaPtr": numpy_port.as_index(optr, nnz, index_bits),
        "rowPtr": numpy_port.as_index(rptr, s, index_bits),
    }
    if kind == "cser":
        out["omegaI"] = numpy_port.as_index(oidx[:s], max(k - 1, 0), index_bits)
        out["mode_index"] = int(mode)
    return out


def encode_cer(values, index_bits="auto", background=None) -> dict:
    return encode(values, "cer", index_bits, background)


def encode_cser(values, index_bits="auto", background=None) -> dict:
    return encode(values, "cser", index_bits, background)


def dot(enc: dict, x) -> np.ndarray:
    """float64 y in the reference loop oracle's summation order (tests/reference_kernels.py:144-203)."""
    xv = np.asarray(x, dtype=np.float64)
    if xv.ndim not in (1, 2):
        raise ValueError("right-hand side must be a vector or a matrix")
    if xv.shape[0] != enc["n"]:
        raise ValueError(f"dimension mismatch: matrix has n={enc['n']}, input has {xv.shape[0]}")
    b = 1 if xv.ndim == 1 else xv.shape[1]
    xc = np.ascontiguousarray(xv.reshape(enc["n"], b))
    y = np.empty((enc["m"], b), dtype=np.float64)
    rp = np.ascontiguousarray(enc["rowPtr"], dtype=np.int64)
    op = np.ascontiguousarray(enc["omegaPtr"], dtype=np.int64)
    col = np.ascontiguousarray(enc["colI"], dtype=np.int64)
    sv = np.ascontiguousarray(numpy_port.segment_values(enc), dtype=np.float64)
    lib().oracle_dot(enc["m"], enc["n"], b, _ptr(rp), _ptr(op), _ptr(col), _ptr(sv),
                     numpy_port.background_of(enc), _ptr(xc), _ptr(y))
    return y[:, 0] if xv.ndim == 1 else y
