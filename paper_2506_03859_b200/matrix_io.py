"""Dense matrix files: the reference's three interchange formats
(/root/reference/proj/src/matrix_io.cpp, declared in include/rsvd/matrix_io.hpp:7-23).

    RawF64             "SKLR" | u32 rows | u32 cols | u32 reserved (0) | rows*cols
                       little-endian f64, column-major            (matrix_io.cpp:141-200)
    MatrixMarket array "%%MatrixMarket matrix array real general", "rows cols",
                       then the entries column-major, one per line  (matrix_io.cpp:40-131)
    PPM (P6)           an h x w image read as the 3h x w matrix [R; G; B] on the
                       [0, 255] scale; 8- or 16-bit (big-endian) samples (:202-301)

Host-side I/O only: this is how A reaches the engine.
Every loader validates like the reference and raises FormatError carrying the
same byte offset the reference reports (the offending byte; the file end for
truncation).  The MatrixMarket reader parses the common all-decimal file with one
vectorised pass and falls back to a cursor that follows the reference's
strtod/strtoll scan exactly whenever the fast pass meets anything unusual, so the
error messages and offsets are the reference's.
"""
from __future__ import annotations

import math
import os
import re
import struct

import numpy as np

from .rsvd import ConfigError, DimensionError, RsvdError

_MAGIC = b"SKLR"
_INT_MAX = 2**31 - 1
_U64_MAX = 2**64 - 1
_TINY = 2.2250738585072014e-308   # smallest normal double


class FormatError(RsvdError, ValueError):
    """Malformed matrix data (rsvd::FormatError, errors.hpp:42-46); `offset` is the byte position."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (at byte {offset})")
        self.msg = msg
        self.offset = offset


# ---- formats by name (matrix_io.cpp:303-322) ------------------------------------
RAW, MATRIX_MARKET, PPM = "rawf64", "matrixmarket", "ppm"


def matrix_format_from_name(name: str) -> str:
    s = name.lower()
    if s in ("mm", "matrixmarket", "mtx"):
        return MATRIX_MARKET
    if s in ("raw", "rawf64"):
        return RAW
    if s == "ppm":
        return PPM
    raise ConfigError("unknown matrix format: " + name)


def matrix_format_name(fmt: str) -> str:
    return matrix_format_from_name(fmt)


# ---- RawF64 -------------------------------------------------------------------
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
    if cols != 0 and rows > (_U64_MAX // 8) // cols:
        raise FormatError("dimension overflow in payload size", 4)
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
    arr = _matrix(a)
    rows, cols = arr.shape
    return _MAGIC + struct.pack("<III", rows, cols, 0) + np.asarray(arr, dtype="<f8").tobytes(order="F")


def _matrix(a) -> np.ndarray:
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("a must be 2-D")
    if arr.shape[0] > _INT_MAX or arr.shape[1] > _INT_MAX:
        raise ValueError("dimensions exceed the format's int range")
    return arr


# ---- MatrixMarket array ------------------------------------------------------------
_MM_BANNER = b"%%MatrixMarket"
_MM_WANT = [b"matrix", b"array", b"real", b"general"]
# strtod's accepted forms (C locale): decimal, hex float, inf/infinity, nan[(chars)]
_STRTOD = re.compile(
    rb"[+-]?(?:(?i:infinity|inf)|(?i:nan)(?:\([0-9A-Za-z_]*\))?"
    rb"|0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?"
    rb"|(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?)")
_STRTOLL = re.compile(rb"[+-]?[0-9]+")
_DECIMAL_TOKENS = re.compile(rb"(?:[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\s+)*")
_WS = b" \t\n\v\f\r"


def _strtod_value(tok: bytes) -> float:
    t = tok.lower()
    body = t.lstrip(b"+-")
    if body.startswith(b"0x"):
        s = t.decode()
        if "p" not in s:
            s += "p0"
        return float.fromhex(s)
    if body.startswith(b"nan"):
        return math.nan
    return float(t)


def _erange(tok: bytes, v: float) -> bool:
    """glibc strtod sets ERANGE on overflow and on underflow (a nonzero decimal that
    rounds to zero or to a subnormal)."""
    body = tok.lower().lstrip(b"+-")
    if body.startswith((b"inf", b"nan")):
        return False
    if math.isinf(v):
        return True
    if v != 0.0:
        return abs(v) < _TINY
    mant = body.split(b"p")[0] if body.startswith(b"0x") else body.split(b"e")[0]
    if body.startswith(b"0x"):
        mant = mant[2:]
    return any(c not in b"0." for c in mant)


class _Cursor:
    """The reference's scan (mm_skip / mm_double / mm_dim, matrix_io.cpp:40-84)."""

    def __init__(self, buf: bytes, pos: int):
        self.b, self.p = buf, pos

    def skip(self):
        b, n = self.b, len(self.b)
        while True:
            while self.p < n and b[self.p] in _WS:
                self.p += 1
            if self.p < n and b[self.p] == 0x25:   # '%'
                nl = b.find(b"\n", self.p)
                self.p = n if nl < 0 else nl
                continue
            return

    def double(self) -> float:
        self.skip()
        if self.p >= len(self.b):
            raise FormatError("unexpected end of file in matrix entries", self.p)
        m = _STRTOD.match(self.b, self.p)
        if not m:
            raise FormatError("expected a real number", self.p)
        v = _strtod_value(m.group())
        if _erange(m.group(), v):
            raise FormatError("number out of range", self.p)
        self.p = m.end()
        return v

    def dim(self, what: str) -> int:
        self.skip()
        at = self.p
        if self.p >= len(self.b):
            raise FormatError("missing " + what, at)
        m = _STRTOLL.match(self.b, self.p)
        if not m:
            raise FormatError("expected " + what, at)
        v = int(m.group())
        if v < 0 or v > _INT_MAX:
            raise FormatError("dimension overflow in " + what, at)
        self.p = m.end()
        return v


def loads_mm(buf: bytes) -> np.ndarray:
    """Parse a MatrixMarket 'matrix array real general' file -> float64 (column-major)."""
    if not buf.startswith(_MM_BANNER):
        raise FormatError("missing %%MatrixMarket banner", 0)
    eol = buf.find(b"\n")
    eol = len(buf) if eol < 0 else eol
    if buf[len(_MM_BANNER):eol].lower().split() != _MM_WANT:
        raise FormatError("unsupported Matrix Market type, need: matrix array real general", 0)
    cur = _Cursor(buf, eol)
    rows = cur.dim("row count")
    cols = cur.dim("column count")
    total = rows * cols
    fast = _mm_entries_fast(buf, cur.p, total)
    if fast is not None:
        return np.asfortranarray(fast.reshape((cols, rows)).T)
    vals = np.empty(total, dtype=np.float64)
    for k in range(total):
        vals[k] = cur.double()
    cur.skip()
    if cur.p != len(buf):
        raise FormatError("trailing data after matrix entries", cur.p)
    return np.asfortranarray(vals.reshape((cols, rows)).T)


def _mm_entries_fast(buf: bytes, pos: int, total: int):
    """All-decimal entries, comments only on their own or after an entry: one
    vectorised conversion.  None -> let the exact cursor decide (and report)."""
    body = re.sub(rb"%[^\n]*", b"", buf[pos:])
    if not body[:1] or body[:1] in _WS:
        pass
    else:
        return None                      # an entry glued to the size line
    text = body + b"\n"
    if _DECIMAL_TOKENS.fullmatch(text.lstrip(_WS)) is None:
        return None
    toks = text.split()
    if len(toks) != total:
        return None
    vals = np.array(toks, dtype=np.float64) if toks else np.empty(0)
    bad = ~np.isfinite(vals) | ((vals != 0) & (np.abs(vals) < _TINY))
    if bad.any():
        return None
    for k in np.flatnonzero(vals == 0):
        if _erange(toks[k], 0.0):
            return None
    return vals


def dumps_mm(a) -> bytes:
    arr = _matrix(a)
    rows, cols = arr.shape
    head = "%%%%MatrixMarket matrix array real general\n%d %d\n" % (rows, cols)
    flat = arr.ravel(order="F")
    return (head + "".join("%.17g\n" % v for v in flat.tolist())).encode()


# ---- PPM (P6) ---------------------------------------------------------------------
def _ppm_int(buf: bytes, p: int, what: str):
    n = len(buf)
    while True:
        while p < n and buf[p] in _WS:
            p += 1
        if p < n and buf[p] == 0x23:   # '#'
            nl = buf.find(b"\n", p)
            p = n if nl < 0 else nl
            continue
        break
    at = p
    if p >= n or not (0x30 <= buf[p] <= 0x39):
        raise FormatError(f"expected {what} in PPM header", at)
    v = 0
    while p < n and 0x30 <= buf[p] <= 0x39:
        v = v * 10 + (buf[p] - 0x30)
        if v > _INT_MAX:
            raise FormatError("dimension overflow in " + what, at)
        p += 1
    return v, at, p


def loads_ppm(buf: bytes) -> np.ndarray:
    """P6 image -> 3h x w float64 matrix [R; G; B], samples scaled by 255 / maxval."""
    if len(buf) < 2 or buf[:2] != b"P6":
        raise FormatError("not a P6 PPM file", 0)
    w, at_w, p = _ppm_int(buf, 2, "width")
    h, at_h, p = _ppm_int(buf, p, "height")
    maxval, at_m, p = _ppm_int(buf, p, "maxval")
    if w < 1:
        raise FormatError("PPM width must be positive", at_w)
    if h < 1:
        raise FormatError("PPM height must be positive", at_h)
    if maxval < 1 or maxval > 65535:
        raise FormatError("PPM maxval out of range", at_m)
    if h * 3 > _INT_MAX:
        raise FormatError("dimension overflow in height", at_h)
    if p >= len(buf) or buf[p] not in _WS:
        raise FormatError("missing separator after maxval", p)
    p += 1
    bps = 1 if maxval < 256 else 2
    need = w * h * 3 * bps
    have = len(buf) - p
    if have < need:
        raise FormatError(f"truncated pixel payload: expected {need} bytes, found {have}", len(buf))
    if have > need:
        raise FormatError("trailing bytes after pixel payload", p + need)
    raw = np.frombuffer(buf, dtype=np.uint8 if bps == 1 else ">u2", count=w * h * 3, offset=p)
    planes = raw.reshape((h, w, 3)).transpose(2, 0, 1).reshape((3 * h, w))
    return np.asfortranarray(planes.astype(np.float64) * (255.0 / maxval))


def dumps_ppm(a) -> bytes:
    arr = _matrix(a)
    if arr.shape[0] % 3 != 0 or arr.shape[0] == 0:
        raise DimensionError("PPM save needs a positive row count divisible by 3")
    h, w = arr.shape[0] // 3, arr.shape[1]
    v = np.where(np.isnan(arr), 0.0, np.clip(arr, 0.0, 255.0))
    fl = np.floor(v)
    r = (fl + (v - fl >= 0.5)).astype(np.uint8)   # lround: halves away from zero
    pix = r.reshape((3, h, w)).transpose(1, 2, 0)
    return b"P6\n%d %d\n255\n" % (w, h) + pix.tobytes()


# ---- files (load_matrix / save_matrix, matrix_io.cpp:314-342) ------------------------
_LOADERS = {RAW: loads_raw, MATRIX_MARKET: loads_mm, PPM: loads_ppm}
_DUMPERS = {RAW: dumps_raw, MATRIX_MARKET: dumps_mm, PPM: dumps_ppm}


def _read(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError:
        raise FormatError(f"cannot open {os.fspath(path)}", 0) from None


def load_matrix(path: str | os.PathLike, fmt: str = RAW) -> np.ndarray:
    return _LOADERS[matrix_format_from_name(fmt)](_read(path))


def save_matrix(a, path: str | os.PathLike, fmt: str = RAW) -> None:
    data = _DUMPERS[matrix_format_from_name(fmt)](a)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError:
        raise FormatError(f"cannot open {os.fspath(path)} for writing", 0) from None


def load_raw(path: str | os.PathLike) -> np.ndarray:
    return loads_raw(_read(path))


def save_raw(path: str | os.PathLike, a) -> None:
    save_matrix(a, path, RAW)


# ---- native RawF64 reads (csrc/rawio.cu): row shards, straight to the device ----------
def _native_check(st: int, off, what: str) -> None:
    if st == 0:
        return
    from . import _native
    msg = _native.lib().fqb_last_error().decode(errors="replace")
    if st == 11:   # FQB_ERR_FORMAT: the reference's FormatError and byte offset
        raise FormatError(msg, int(off.value))
    from .rsvd import _raise
    _raise(st, f"{what}: {msg}")


def raw_header(path: str | os.PathLike) -> tuple[int, int]:
    """(rows, cols) of a RawF64 file, validated like the reference's loader (FormatError)."""
    import ctypes as C
    from . import _native
    r, c, off = C.c_int64(), C.c_int64(), C.c_int64()
    st = _native.lib().fqb_raw_header(os.fsencode(path), C.byref(r), C.byref(c), C.byref(off))
    _native_check(st, off, "fqb_raw_header")
    return r.value, c.value


def load_raw_rows(path: str | os.PathLike, row0: int = 0, rows: int | None = None, engine=None):
    """Rows [row0, row0 + rows) of a RawF64 file (a rank's row shard; default all rows).

    engine=None: a host float64 array (Fortran order), read by parallel preads.
    engine=Engine: a column-major torch tensor on that engine's device, uploaded through
    pinned staging panels overlapped with the reads (fqb_load_raw_rows)."""
    import ctypes as C
    from . import _native
    m, n = raw_header(path)
    rows = m - row0 if rows is None else rows
    off = C.c_int64()
    if engine is None:
        out = np.empty((n, rows), dtype=np.float64).T    # column-major rows x n
        st = _native.lib().fqb_load_raw_rows(None, os.fsencode(path), row0, rows, out.ctypes.data, max(rows, 1), 0,
                                             C.byref(off))
        _native_check(st, off, "fqb_load_raw_rows")
        return out
    import torch
    out = torch.empty((n, rows), dtype=torch.float64, device=f"cuda:{engine.device}").t()
    st = _native.lib().fqb_load_raw_rows(engine._h, os.fsencode(path), row0, rows, out.data_ptr(), max(rows, 1), 1,
                                         C.byref(off))
    _native_check(st, off, "fqb_load_raw_rows")
    return out
