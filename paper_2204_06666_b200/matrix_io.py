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
