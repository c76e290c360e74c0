"""B200-native CER/CSER conversion and dot product (arXiv 1805.10692).

Drop-in for the hot path of the reference package ``lemt``
(``lemt/__init__.py:24-41``): the same names and signatures for the
CER/CSER encoders and dot products, backed by hand-written sm_100a kernels
in ``libcerdot.so`` (C ABI: ``include/cerdot.h``).  There is no CPU
fallback: the device calls raise ``RuntimeError`` without CUDA.
"""

from .matrices import DenseMatrix, Vector
from .formats import (
    CerMatrix,
    CserMatrix,
    FormatError,
    array_bytes,
    decode,
    encode_cer,
    encode_cser,
    encode_pair,
    entry_count,
    index_bitwidth,
    storage_bits,
    validate,
)
from .io import IoFormatError, read_matrix, write_matrix
from .kernels import OpTrace, dot, dot_cer, dot_cser, dot_device, row_trace, trace_cer, trace_cser, trace_of

__version__ = "0.1.0"

__all__ = [
    "DenseMatrix", "Vector", "CerMatrix", "CserMatrix", "FormatError", "array_bytes", "decode", "validate", "encode_cer",
    "encode_cser", "encode_pair", "entry_count", "index_bitwidth", "storage_bits", "OpTrace", "dot", "dot_cer", "dot_cser",
    "dot_device", "row_trace", "trace_cer", "trace_cser", "trace_of", "IoFormatError", "read_matrix",
    "write_matrix",
]
