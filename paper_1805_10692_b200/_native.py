"""ctypes binding of libcerdot (include/cerdot.h).

The library is the product: there is no CPU fallback.  Loading fails loudly
when the shared object is missing, and every call that needs a GPU fails
loudly when CUDA is unavailable.
"""

from __future__ import annotations

import ctypes
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.environ.get("CERDOT_LIB") or os.path.join(PKG, "_lib", "libcerdot.so")
HEADER = os.path.join(ROOT, "include", "cerdot.h")

OK, E_VALUE, E_TYPE, E_INDEX, E_CUDA, E_UNSUPPORTED, E_WORKSPACE, E_FORMAT = range(8)
CER, CSER = 0, 1
F32, F64 = 0, 1
FAST_K = 2048


class CerdotFormatError(ctypes.Structure):  # cerdot_format_error
    _fields_ = [("check", ctypes.c_int32), ("offset", ctypes.c_int64), ("value", ctypes.c_int64)]


class CerdotMatrix(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("mode_index", ctypes.c_int32),
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("segments", ctypes.c_int64),
        ("omega", ctypes.c_void_p),
        ("col_index", ctypes.c_void_p),
        ("omega_ptr", ctypes.c_void_p),
        ("row_ptr", ctypes.c_void_p),
        ("omega_index", ctypes.c_void_p),
        ("col_bits", ctypes.c_int32),
        ("omega_ptr_bits", ctypes.c_int32),
        ("row_ptr_bits", ctypes.c_int32),
        ("omega_index_bits", ctypes.c_int32),
        ("background", ctypes.c_double),
        ("max_row_nnz", ctypes.c_int64),
        ("max_row_segments", ctypes.c_int64),
        ("row_entry", ctypes.c_void_p),
        ("tile_rows", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
        ("tile_ptr", ctypes.c_void_p),
        ("tile_rec", ctypes.c_void_p),
    ]


class CerdotEncodeInfo(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("segments_cer", ctypes.c_int64),
        ("segments_cser", ctypes.c_int64),
        ("mode_index", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("background", ctypes.c_double),
        ("workspace_bytes", ctypes.c_size_t),
        ("max_row_nnz", ctypes.c_int64),
        ("max_row_segments_cer", ctypes.c_int64),
        ("max_row_segments_cser", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_SIGNATURES = {
    "cerdot_abi_version": (ctypes.c_int, []),
    "cerdot_last_error": (ctypes.c_char_p, []),
    "cerdot_index_bitwidth": (_I32, [_I64]),
    "cerdot_encode_workspace_bytes": (_SZ, [_I64, _I64]),
    "cerdot_encode_plan": (ctypes.c_int, [_P, _I32, _I64, _I64, _I64, _I32, ctypes.c_double, _P, _SZ,
                                          ctypes.POINTER(CerdotEncodeInfo), _P]),
    "cerdot_encode_fill": (ctypes.c_int, [ctypes.POINTER(CerdotEncodeInfo), _I32, _P, _SZ, _P, _P, _I32, _P, _I32,
                                          _P, _I32, _P, _I32, _P]),
    "cerdot_dot_workspace_bytes": (_SZ, [ctypes.POINTER(CerdotMatrix), _I64]),
    "cerdot_dot": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _I64, _P, _I64, _P, _SZ, _P]),
    "cerdot_validate_workspace_bytes": (_SZ, [ctypes.POINTER(CerdotMatrix)]),
    "cerdot_validate": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), ctypes.POINTER(CerdotFormatError), _P, _SZ,
                                       _P]),
    "cerdot_decode": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _P]),
    "cerdot_trace_counts": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _P, _P]),
    "cerdot_lemx_unpack": (ctypes.c_int, [_P, _I32, _I64, _I64, _P, _P, _I32, _P, _P]),
    "cerdot_dot_peers": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _I64, _P, _I64, _P, _I32, _I64, _P,
                                        _SZ, _P]),
    "cerdot_dot_cer": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _I64, _P, _I64, _P, _SZ, _P]),
    "cerdot_dot_cser": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _I64, _P, _I64, _P, _SZ, _P]),
    "cerdot_dot_host_workspace_bytes": (_SZ, [ctypes.POINTER(CerdotMatrix), _I64]),
    "cerdot_dot_host": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _I64, _I64, _P, _I64, _P, _SZ, _P]),
    "cerdot_row_entries": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _P, _P]),
    "cerdot_shard_plan": (ctypes.c_int, [_P, _I32, _P, _I32, _I32, _I32, _I64, _I32, ctypes.POINTER(ctypes.c_int64)]),
    "cerdot_tile_view_rows": (_I32, [ctypes.POINTER(CerdotMatrix), _I64]),
    "cerdot_tile_view_workspace_bytes": (_SZ, [ctypes.POINTER(CerdotMatrix), _I32]),
    "cerdot_tile_view_build": (ctypes.c_int, [ctypes.POINTER(CerdotMatrix), _I32, _P, _P, _P, _SZ, _P]),
    "cerdot_set_kernel_path": (_I32, [_I32, _I32]),
    "cerdot_synth_choice": (ctypes.c_int, [_P, _P, ctypes.c_uint64, _P, _P, _I32, _I64, _P, _P]),
}

# cerdot_path_op
PATH_OPS = {"matvec": 0, "matmat": 1, "matvec_nt": 2, "matmat_depth": 3, "trace": 4, "matmat_split": 5, "matmat_tile": 6}
# named kernel choices per op (the integers of include/cerdot.h)
PATH_NAMES = {"matvec": {"auto": 0, "window": 1, "tile": 2, "run": 3, "stream": 4, "row": 5},
              "matmat": {"auto": 0, "flat": 1, "segment": 2, "tiled": 3, "tiled_frag": 4}}

_lib = None


def header_functions() -> list[str]:
    """Every function the public header declares (used by the export test)."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(cerdot_\w+)\s*\(", text, flags=re.M)))


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libcerdot.so not found at {LIB_PATH}; build it with `python -m paper_1805_10692_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            if os.environ.get("CERDOT_LIB") and not hasattr(L, name):
                continue  # A/B timing against an older build (tools/ab_build.sh): newer entry points absent
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.cerdot_abi_version() != 3:
            raise ImportError("libcerdot ABI version mismatch")
        _lib = L
    return _lib


class force_path:
    """Context manager: pin a kernel choice (cerdot_set_kernel_path) for A/B timing and parity tests,
    e.g. ``with force_path("matvec", "run"): ...``.  Process-wide; restores the previous value."""

    def __init__(self, op: str, path):
        self.op = PATH_OPS[op]
        self.path = PATH_NAMES.get(op, {}).get(path, path) if isinstance(path, str) else int(path)
        self.prev = None

    def __enter__(self):
        self.prev = lib().cerdot_set_kernel_path(self.op, int(self.path))
        return self

    def __exit__(self, *exc):
        lib().cerdot_set_kernel_path(self.op, self.prev)
        return False


def last_error() -> str:
    msg = lib().cerdot_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Map a status code onto the reference's exception types."""
    if status == OK:
        return
    msg = last_error()
    if status == E_VALUE:
        raise ValueError(msg)
    if status == E_TYPE:
        raise TypeError(msg)
    if status == E_INDEX:
        raise IndexError(msg)
    raise RuntimeError(f"libcerdot: {msg} (status {status})")
