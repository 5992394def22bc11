"""HNMW binary matrices (reference io.py:19-49): magic 'HNMW', u32 version=1, u32 rows,
u32 cols, then rows*cols little-endian float32, row-major.  Host I/O only."""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import FormatError
from .model import as_values

_HDR = struct.Struct("<4sIII")


def write_hnmw(path, matrix) -> None:
    v = as_values(matrix)
    if v.ndim != 2:
        raise FormatError(f"HNMW stores 2-D matrices, got shape {v.shape}")
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(b"HNMW", 1, v.shape[0], v.shape[1]))
        fh.write(np.ascontiguousarray(v, dtype="<f4").tobytes())


def read_hnmw(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if len(raw) < _HDR.size:
        raise FormatError(f"{path}: truncated header")
    magic, version, rows, cols = _HDR.unpack_from(raw)
    if magic != b"HNMW":
        raise FormatError(f"{path}: bad magic {magic!r}")
    if version != 1:
        raise FormatError(f"{path}: unsupported version {version}")
    if len(raw) != _HDR.size + 4 * rows * cols:
        raise FormatError(f"{path}: expected {_HDR.size + 4 * rows * cols} bytes, found {len(raw)}")
    return np.frombuffer(raw, dtype="<f4", offset=_HDR.size).reshape(rows, cols).astype(np.float64)
