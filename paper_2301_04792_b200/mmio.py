"""Matrix Market coordinate-format reader and writer (reference mmio.py).

Supported inputs: banner ``%%MatrixMarket matrix coordinate <field> <symmetry>``
with field in {real, integer, pattern} and symmetry in {general, symmetric}.
Pattern entries get value 1.0; symmetric files expand off-diagonal entries to
both triangles. Indices are 1-based on disk and 0-based in memory.

Parsing runs in the native library (lw_mm_parse_header / lw_mm_parse_entries,
include/lw_b200.h): multi-threaded over line-aligned chunks of the raw bytes,
with the reference's accepted syntax, error precedence and messages.
"""

from __future__ import annotations

import ctypes
import io
from os import PathLike

import numpy as np

from . import _lib
from .sparse import CooMatrix

__all__ = ["MatrixMarketError", "parse_matrix_market", "load_matrix_market",
           "write_matrix_market"]

_ERRLEN = 512


class MatrixMarketError(ValueError):
    """Raised for any malformed or unsupported Matrix Market input."""


def _parse_bytes(buf, threads: int = 0) -> CooMatrix:
    lib = _lib.load()
    n = len(buf)
    cbuf = bytes(buf)
    err = ctypes.create_string_buffer(_ERRLEN)
    h = _lib.LwMmHeader()
    rc = lib.lw_mm_parse_header(cbuf, n, ctypes.byref(h), err, _ERRLEN)
    if rc == _lib.LW_E_FORMAT:
        raise MatrixMarketError(err.value.decode("utf-8", "replace"))
    _lib.check(rc, "lw_mm_parse_header")
    cap = h.entries * (2 if h.symmetric else 1)
    row = np.empty(cap, dtype=np.int64)
    col = np.empty(cap, dtype=np.int64)
    val = np.empty(cap, dtype=np.float64)
    count = ctypes.c_int64(0)

    def ptr(a):
        return a.ctypes.data if a.size else None

    rc = lib.lw_mm_parse_entries(cbuf, n, ctypes.byref(h), ptr(row),
                                 ptr(col), ptr(val), cap, ctypes.byref(count), threads, err,
                                 _ERRLEN)
    if rc == _lib.LW_E_FORMAT:
        raise MatrixMarketError(err.value.decode("utf-8", "replace"))
    _lib.check(rc, "lw_mm_parse_entries")
    k = count.value
    return CooMatrix(int(h.rows), int(h.cols), row[:k], col[:k], val[:k])


def parse_matrix_market(source, threads: int = 0) -> CooMatrix:
    """Parse Matrix Market text (a string, bytes, or a file object) into a CooMatrix."""
    if isinstance(source, str):
        data = source.encode("utf-8", "surrogateescape")
    elif isinstance(source, (bytes, bytearray)):
        data = bytes(source)
    elif isinstance(source, io.TextIOBase) or hasattr(source, "read"):
        text = source.read()
        data = text.encode("utf-8", "surrogateescape") if isinstance(text, str) else bytes(text)
    else:
        raise TypeError("source must be str, bytes or a file object")
    return _parse_bytes(data, threads)


def load_matrix_market(path: str | PathLike, threads: int = 0) -> CooMatrix:
    """Read a .mtx file and parse its bytes with the native reader."""
    with open(path, "rb") as fh:
        return _parse_bytes(fh.read(), threads)


def write_matrix_market(coo: CooMatrix, field: str = "real") -> str:
    """Serialize a CooMatrix in coordinate/general form (1-based indices)."""
    if field not in ("real", "integer", "pattern"):
        raise ValueError(f"unsupported field {field!r}")
    out = [f"%%MatrixMarket matrix coordinate {field} general", f"{coo.rows} {coo.cols} {coo.nnz}"]
    if field == "pattern":
        out += [f"{i + 1} {j + 1}" for i, j in zip(coo.row.tolist(), coo.col.tolist())]
    elif field == "integer":
        out += [f"{i + 1} {j + 1} {int(v)}" for i, j, v in coo.entries()]
    else:
        out += [f"{i + 1} {j + 1} {v!r}" for i, j, v in coo.entries()]
    return "\n".join(out) + "\n"
