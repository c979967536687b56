"""Boundary input types (reference matrix_io.py:30-108) and the COO<->CSR
conversions that feed the cuSPARSE comparator (matrix_io.py:255-273).

Same field names, dtypes, validation and error wording as the reference so
a `CooMatrix` built for the reference works here unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; the message names the offending line."""


class UnsupportedFormatError(MatrixMarketError):
    """Valid Matrix Market input that this library deliberately rejects."""


class ContainerError(ValueError):
    """Corrupt, truncated, or incompatible .ehyb container."""


@dataclass(eq=False)
class CooMatrix:
    """Coordinate-format sparse matrix: int64 rows/cols, float64 values,
    0-based, bounds-validated on construction (matrix_io.py:30-69)."""

    n_rows: int
    n_cols: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.rows = np.asarray(self.rows, dtype=np.int64)
        self.cols = np.asarray(self.cols, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if not (self.rows.shape == self.cols.shape == self.values.shape):
            raise ValueError("rows, cols and values must have equal length")
        if self.rows.ndim != 1:
            raise ValueError("entry arrays must be one-dimensional")
        if self.rows.size:
            if self.rows.min() < 0 or self.rows.max() >= self.n_rows:
                raise ValueError("row index out of bounds")
            if self.cols.min() < 0 or self.cols.max() >= self.n_cols:
                raise ValueError("column index out of bounds")

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def is_square(self) -> bool:
        return self.n_rows == self.n_cols

    def entry_set(self) -> set:
        return set(zip(self.rows.tolist(), self.cols.tolist(), self.values.tolist()))


@dataclass(eq=False)
class CsrMatrix:
    """Compressed sparse rows; columns strictly increasing within a row
    (matrix_io.py:72-108)."""

    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.asarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(self.col_idx, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.row_ptr.size != self.n_rows + 1:
            raise ValueError("row_ptr must have length n_rows + 1")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != self.values.size:
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if np.any(self.row_ptr[1:] < self.row_ptr[:-1]):
            raise ValueError("row_ptr must be non-decreasing")
        if self.col_idx.size != self.values.size:
            raise ValueError("col_idx and values must have equal length")
        nnz = self.values.size
        if nnz > 1:
            row_of = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
            same_row = row_of[1:] == row_of[:-1]
            if np.any(same_row & (self.col_idx[1:] <= self.col_idx[:-1])):
                raise ValueError("col_idx must be strictly increasing within each row")

    @property
    def nnz(self) -> int:
        return int(self.values.size)


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Entries sorted by (row, col); duplicates rejected (matrix_io.py:255-268)."""
    order = np.lexsort((m.cols, m.rows))
    r, c, v = m.rows[order], m.cols[order], m.values[order]
    if r.size > 1 and np.any((r[1:] == r[:-1]) & (c[1:] == c[:-1])):
        raise ValueError("duplicate (row, col) entries")
    row_ptr = np.zeros(m.n_rows + 1, dtype=np.int64)
    if r.size:
        np.cumsum(np.bincount(r, minlength=m.n_rows), out=row_ptr[1:])
    return CsrMatrix(m.n_rows, m.n_cols, row_ptr, c, v)


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    rows = np.repeat(np.arange(m.n_rows, dtype=np.int64), np.diff(m.row_ptr))
    return CooMatrix(m.n_rows, m.n_cols, rows, m.col_idx.copy(), m.values.copy())


# --------------------------------------------------------------------------
# .ehyb container (reference matrix_io.py:276-474): persists an assembled
# EhybMatrix so preprocessing is paid once (SPEC.md amortisation argument).
#   "EHYB" | version u32 | tau u32 | payload | crc32(payload) u32, little-endian;
#   payload = every field as (u64 byte length, bytes): 7 u64 scalars, then
#   the tables as i32 and the bodies as u16 / u32 / f32|f64.
# --------------------------------------------------------------------------

import struct as _struct
import zlib as _zlib

_MAGIC = b"EHYB"
_VERSION = 1
_SCALARS = ("dimension", "padded_dimension", "k", "n_parts", "vec_cache_size", "warp_size",
            "n_er_rows")
# (field, dtype) in payload order; "val" resolves to f32 / f64 by tau
_ARRAYS = (("reorder_table", "<i4"), ("inverse_table", "<i4"), ("arrange_table", "<i4"),
           ("y_idx_er", "<i4"), ("part_boundary", "<i4"), ("position_ell", "<i4"),
           ("width_ell", "<i4"), ("ell_row_widths", "<i4"), ("col_ell", "<u2"),
           ("val_ell", "val"), ("position_er", "<i4"), ("width_er", "<i4"),
           ("er_row_widths", "<i4"), ("col_er", "<u4"), ("val_er", "val"))


def _field_source(e, name):
    if name in ("reorder_table", "inverse_table", "arrange_table", "y_idx_er"):
        return getattr(e.plan, name)
    return getattr(e, name)


def write_ehyb_container(e, sink) -> None:
    """Serialise an EhybMatrix; read_ehyb_container inverts it bit-exactly."""
    tau = e.params.tau
    vdt = "<f4" if tau == 4 else "<f8"
    scal = dict(dimension=e.dimension, padded_dimension=e.padded_dimension, k=e.params.k,
                n_parts=e.params.n_parts, vec_cache_size=e.params.vec_cache_size,
                warp_size=e.params.warp_size, n_er_rows=e.plan.n_er_rows)
    chunks = []
    for name in _SCALARS:
        chunks.append(_struct.pack("<QQ", 8, int(scal[name])))
    for name, dt in _ARRAYS:
        raw = np.ascontiguousarray(_field_source(e, name), vdt if dt == "val" else dt).tobytes()
        chunks.append(_struct.pack("<Q", len(raw)))
        chunks.append(raw)
    payload = b"".join(chunks)
    blob = (_MAGIC + _struct.pack("<II", _VERSION, tau) + payload
            + _struct.pack("<I", _zlib.crc32(payload) & 0xFFFFFFFF))
    if isinstance(sink, (str, bytes)) or hasattr(sink, "__fspath__"):
        with open(sink, "wb") as fh:
            fh.write(blob)
    else:
        sink.write(blob)


def read_ehyb_container(source):
    """Deserialise a .ehyb container (CRC checked before any field is read);
    raises ContainerError on bad magic / version / tag, truncation, CRC or
    inconsistent contents."""
    from .format import EhybMatrix, EhybParams, ReorderPlan

    if isinstance(source, (bytes, bytearray)):
        blob = bytes(source)
    elif isinstance(source, str) or hasattr(source, "__fspath__"):
        with open(source, "rb") as fh:
            blob = fh.read()
    else:
        blob = source.read()
    if len(blob) < 16:
        raise ContainerError("truncated stream: missing header")
    if blob[:4] != _MAGIC:
        raise ContainerError("bad magic: not an EHYB container")
    version, tau = _struct.unpack_from("<II", blob, 4)
    if version != _VERSION:
        raise ContainerError(f"unsupported container version {version}")
    if tau not in (4, 8):
        raise ContainerError(f"invalid precision tag {tau}")
    view = memoryview(blob)[12:-4]
    (crc,) = _struct.unpack_from("<I", blob, len(blob) - 4)
    if (_zlib.crc32(view) & 0xFFFFFFFF) != crc:
        raise ContainerError("checksum failure: payload does not match CRC32")
    off = 0

    def take(what):
        nonlocal off
        if off + 8 > len(view):
            raise ContainerError(f"truncated stream while reading {what} length")
        (ln,) = _struct.unpack_from("<Q", view, off)
        off += 8
        if off + ln > len(view):
            raise ContainerError(f"truncated stream while reading {what}")
        out = view[off: off + ln]
        off += ln
        return out

    sc = {}
    for name in _SCALARS:
        raw = take(name)
        if len(raw) != 8:
            raise ContainerError(f"bad scalar length for {name}")
        (sc[name],) = _struct.unpack("<Q", raw)
    arrs = {}
    vdt = np.dtype("<f4" if tau == 4 else "<f8")
    for name, dt in _ARRAYS:
        d = vdt if dt == "val" else np.dtype(dt)
        raw = take(name)
        if len(raw) % d.itemsize:
            raise ContainerError(f"array length not a multiple of item size for {name}")
        arrs[name] = np.frombuffer(raw, dtype=d).copy()
    if off != len(view):
        raise ContainerError("trailing bytes after last field")
    try:
        params = EhybParams(k=int(sc["k"]), n_parts=int(sc["n_parts"]),
                            vec_cache_size=int(sc["vec_cache_size"]), tau=int(tau),
                            warp_size=int(sc["warp_size"]))
        plan = ReorderPlan(reorder_table=arrs["reorder_table"],
                           inverse_table=arrs["inverse_table"],
                           arrange_table=arrs["arrange_table"], y_idx_er=arrs["y_idx_er"],
                           n_er_rows=int(sc["n_er_rows"]), dimension=int(sc["dimension"]),
                           padded_dimension=int(sc["padded_dimension"]))
        e = EhybMatrix(params=params, plan=plan, dimension=int(sc["dimension"]),
                       padded_dimension=int(sc["padded_dimension"]),
                       **{k: arrs[k] for k in ("val_ell", "col_ell", "position_ell", "width_ell",
                                               "part_boundary", "ell_row_widths", "val_er",
                                               "col_er", "position_er", "width_er",
                                               "er_row_widths")})
        e.check()
    except ValueError as exc:
        raise ContainerError(f"inconsistent container contents: {exc}") from exc
    return e
