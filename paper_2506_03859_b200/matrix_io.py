"""RawF64 matrix files, the reference's interchange format (load_raw / save_raw,
/root/reference/proj/src/matrix_io.cpp:141-200):

    "SKLR" | u32 rows | u32 cols | u32 reserved (0) | rows*cols little-endian f64, column-major

Host-side I/O only (the way A reaches the engine).  The
loader validates like the reference: magic, 16-byte header, payload size exact
(no truncation, no trailing bytes), dimensions within int range.
"""
from __future__ import annotations

import os
import struct

import numpy as np

from .rsvd import RsvdError

_MAGIC = b"SKLR"
_INT_MAX = 2**31 - 1


class FormatError(RsvdError, ValueError):
    """Malformed RawF64 data (rsvd::FormatError); `offset` is the byte position."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (at byte {offset})")
        self.offset = offset


def loads_raw(buf: bytes) -> np.ndarray:
    """Parse RawF64 bytes -> float64 array in Fortran (column-major) order."""
    if len(buf) < 16:
        raise FormatError("truncated header, need 16 bytes", len(buf))
    if buf[:4] != _MAGIC:
        raise FormatError("bad magic, expected SKLR", 0)
    rows, cols, _reserved = struct.unpack_from("<III", buf, 4)
    if rows > _INT_MAX:
        raise FormatError("dimension overflow in row count", 4)
    if cols > _INT_MAX:
        raise FormatError("dimension overflow in column count", 8)
    need = rows * cols * 8
    have = len(buf) - 16
    if have < need:
        raise FormatError(f"truncated payload: expected {need} bytes, found {have}", len(buf))
    if have > need:
        raise FormatError("trailing bytes after payload", 16 + need)
    flat = np.frombuffer(buf, dtype="<f8", count=rows * cols, offset=16)
    return np.asfortranarray(flat.reshape((cols, rows)).T.astype(np.float64, copy=True))


def dumps_raw(a) -> bytes:
    """float64 matrix -> RawF64 bytes (reserved word 0)."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("a must be 2-D")
    rows, cols = arr.shape
    if rows > _INT_MAX or cols > _INT_MAX:
        raise ValueError("dimensions exceed the format's int range")
    return _MAGIC + struct.pack("<III", rows, cols, 0) + np.asarray(arr, dtype="<f8").tobytes(order="F")


def load_raw(path: str | os.PathLike) -> np.ndarray:
    with open(path, "rb") as f:
        return loads_raw(f.read())


def save_raw(path: str | os.PathLike, a) -> None:
    with open(path, "wb") as f:
        f.write(dumps_raw(a))
