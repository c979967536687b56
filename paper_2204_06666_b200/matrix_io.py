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


# --------------------------------------------------------------------------
# Matrix Market text (reference matrix_io.py:111-252), parsed with numpy
# --------------------------------------------------------------------------

def _mm_text(source) -> str:
    import os

    if isinstance(source, (str, os.PathLike)):
        with open(source, "rb") as fh:
            return fh.read().decode("latin-1")
    if isinstance(source, (bytes, bytearray)):
        return bytes(source).decode("latin-1")
    data = source.read()
    return data.decode("latin-1") if isinstance(data, bytes) else data


def parse_matrix_market(source) -> CooMatrix:
    """Matrix Market "coordinate" text -> CooMatrix (reference contract,
    matrix_io.py:123-231): path, bytes or file object; symmetric input
    mirrored to general storage, pattern entries valued 1.0, 1-based indices
    made 0-based, duplicates summed (entries end up sorted by (row, col)).
    Errors name the offending line: MatrixMarketError for malformed input,
    UnsupportedFormatError for complex / array / other symmetries.

    Entry lines are converted in one vectorised pass; only malformed input
    falls back to a line-by-line scan to name the line."""
    lines = _mm_text(source).splitlines()
    if not lines:
        raise MatrixMarketError("line 1: empty input")
    head = lines[0].strip().split()
    if len(head) != 5 or head[0].lower() != "%%matrixmarket":
        raise MatrixMarketError("line 1: malformed Matrix Market header")
    obj, fmt, field, symmetry = (t.lower() for t in head[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"line 1: unsupported object {obj!r}")
    if fmt == "array":
        raise UnsupportedFormatError("line 1: dense 'array' files are not supported")
    if fmt != "coordinate":
        raise MatrixMarketError(f"line 1: unknown format {fmt!r}")
    if field == "complex":
        raise UnsupportedFormatError("line 1: complex-valued matrices are not supported")
    if field not in ("real", "integer", "pattern"):
        raise MatrixMarketError(f"line 1: unknown field {field!r}")
    if symmetry not in ("general", "symmetric"):
        raise UnsupportedFormatError(f"line 1: unsupported symmetry {symmetry!r}")
    i = 1
    while True:
        if i >= len(lines):
            raise MatrixMarketError(f"line {i + 1}: missing size line")
        text = lines[i].strip()
        i += 1
        if text and not text.startswith("%"):
            break
    tok = text.split()
    if len(tok) != 3:
        raise MatrixMarketError(f"line {i}: size line must be 'rows cols nnz'")
    try:
        n_rows, n_cols, n_decl = (int(t) for t in tok)
    except ValueError:
        raise MatrixMarketError(f"line {i}: size line must contain integers") from None
    if min(n_rows, n_cols, n_decl) < 0:
        raise MatrixMarketError(f"line {i}: negative size")
    pattern = field == "pattern"
    want = 2 if pattern else 3
    body = [(k + 1, ln) for k, ln in enumerate(lines[i:], start=i)
            if ln.strip() and not ln.lstrip().startswith("%")]
    try:
        if len(body) != n_decl:
            raise ValueError
        rows = np.empty(n_decl, np.int64)
        cols = np.empty(n_decl, np.int64)
        vals = np.ones(n_decl, np.float64)
        if n_decl:
            fields = [ln.split() for _, ln in body]
            if min(len(f) for f in fields) < want:
                raise ValueError
            rows[:] = np.array([f[0] for f in fields], dtype=np.int64)
            cols[:] = np.array([f[1] for f in fields], dtype=np.int64)
            if not pattern:
                vals[:] = np.array([f[2] for f in fields], dtype=np.float64)
            if (rows.min() < 1 or rows.max() > n_rows or cols.min() < 1
                    or cols.max() > n_cols):
                raise ValueError
    except (ValueError, OverflowError):
        _mm_locate_error(body, n_rows, n_cols, n_decl, want, pattern, len(lines))
        raise MatrixMarketError("malformed entries") from None
    r, c, v = rows - 1, cols - 1, vals
    if symmetry == "symmetric":
        off = r != c
        r, c, v = (np.concatenate([r, c[off]]), np.concatenate([c, r[off]]),
                   np.concatenate([v, v[off]]))
    if r.size:
        key = r * np.int64(max(n_cols, 1)) + c
        uniq, inverse = np.unique(key, return_inverse=True)
        summed = np.zeros(uniq.size, np.float64)
        np.add.at(summed, inverse, v)
        r, c, v = uniq // max(n_cols, 1), uniq % max(n_cols, 1), summed
    return CooMatrix(n_rows, n_cols, r, c, v)


def _mm_locate_error(body, n_rows, n_cols, n_decl, want, pattern, n_lines):
    """Line-by-line scan reproducing the reference's error messages."""
    for seen, (lineno, ln) in enumerate(body):
        if seen == n_decl:
            raise MatrixMarketError(f"line {lineno}: extra entry beyond the declared {n_decl}")
        t = ln.split()
        if len(t) < want:
            raise MatrixMarketError(f"line {lineno}: expected {want} fields per entry")
        try:
            a, b = int(t[0]), int(t[1])
            if not pattern:
                float(t[2])
        except ValueError:
            raise MatrixMarketError(f"line {lineno}: malformed entry") from None
        if not (1 <= a <= n_rows and 1 <= b <= n_cols):
            raise MatrixMarketError(f"line {lineno}: index out of declared bounds")
    if len(body) != n_decl:
        raise MatrixMarketError(f"line {n_lines}: expected {n_decl} entries, found {len(body)}")


def write_matrix_market(m: CooMatrix, sink) -> None:
    """CooMatrix -> Matrix Market coordinate/real/general text, entries in
    (row, col) order, values with 17 significant digits (matrix_io.py:234-252)."""
    import os

    order = np.lexsort((m.cols, m.rows))
    body = "\n".join(f"{a} {b} {x:.17g}" for a, b, x in
                     zip(m.rows[order] + 1, m.cols[order] + 1, m.values[order]))
    text = (f"%%MatrixMarket matrix coordinate real general\n{m.n_rows} {m.n_cols} {m.nnz}\n"
            + (body + "\n" if m.nnz else ""))
    if isinstance(sink, (str, os.PathLike)):
        with open(sink, "w") as fh:
            fh.write(text)
    else:
        try:
            sink.write(text)
        except TypeError:
            sink.write(text.encode("ascii"))
