"""Host-side CSC container used at the API boundary.

Mirrors the reference container (pkg/src/qsocp/sparse.py:17-116): int64
index arrays, float64 values, explicit zeros preserved, duplicates summed by
``csc_from_triplets``.  Only what the GPU path needs on the host lives here;
all products run on the device (csrc/spmv.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import BadSparseStructure, IndexOutOfRange

_I = np.int64
_F = np.float64


@dataclass
class SparseMatrixCSC:
    rows: int
    cols: int
    col_pointers: np.ndarray
    row_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_pointers[self.cols])

    def copy(self) -> "SparseMatrixCSC":
        return SparseMatrixCSC(self.rows, self.cols, self.col_pointers.copy(),
                               self.row_indices.copy(), self.values.copy())

    def column_of_entry(self) -> np.ndarray:
        """Column index of every stored entry (length nnz)."""
        return np.repeat(np.arange(self.cols, dtype=_I), np.diff(self.col_pointers))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols))
        np.add.at(out, (self.row_indices, self.column_of_entry()), self.values)
        return out

    def to_dense_symmetric(self) -> np.ndarray:
        up = self.to_dense()
        return up + up.T - np.diag(np.diag(up))


def empty_csc(rows: int, cols: int) -> SparseMatrixCSC:
    return SparseMatrixCSC(rows, cols, np.zeros(cols + 1, _I), np.zeros(0, _I), np.zeros(0, _F))


def check_csc(M: SparseMatrixCSC) -> None:
    """Vectorised CSC invariant check (reference: sparse.py:53-69)."""
    cp = np.asarray(M.col_pointers)
    if cp.shape != (M.cols + 1,) or cp[0] != 0:
        raise BadSparseStructure("column pointer array must have length cols+1 and start at 0")
    width = np.diff(cp)
    if np.any(width < 0):
        raise BadSparseStructure("column pointers must be nondecreasing")
    nnz = int(cp[-1])
    if len(M.row_indices) != nnz or len(M.values) != nnz:
        raise BadSparseStructure("index/value arrays disagree with col_pointers[-1]")
    if nnz == 0:
        return
    ri = np.asarray(M.row_indices)
    if ri.min() < 0 or ri.max() >= M.rows:
        raise BadSparseStructure("row index out of range")
    # strictly increasing inside every column: a non-positive step is only
    # allowed where a new column starts
    step_ok = np.diff(ri) > 0
    starts = cp[1:-1]
    starts = starts[(starts > 0) & (starts < nnz)]
    step_ok[starts - 1] = True
    if not np.all(step_ok):
        j = int(np.searchsorted(cp, np.flatnonzero(~step_ok)[0], side="right") - 1)
        raise BadSparseStructure(f"row indices not strictly increasing in column {j}")


def csc_from_triplets(rows: int, cols: int, triplets) -> SparseMatrixCSC:
    """(row, col, value) triplets -> CSC; duplicates summed, zeros kept.

    Semantics of reference sparse.py:83-116 (the resulting pattern is the union
    of the triplet positions, duplicates are added in input order).
    """
    if isinstance(triplets, tuple) and len(triplets) == 3:
        r, c, v = (np.asarray(a) for a in triplets)
    else:
        t = list(triplets)
        r = np.array([e[0] for e in t])
        c = np.array([e[1] for e in t])
        v = np.array([e[2] for e in t])
    r = r.astype(_I, copy=False).reshape(-1)
    c = c.astype(_I, copy=False).reshape(-1)
    v = v.astype(_F, copy=False).reshape(-1)
    if r.size and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= cols):
        raise IndexOutOfRange("triplet index outside declared shape")
    key = c * _I(max(rows, 1)) + r
    order = np.argsort(key, kind="stable")
    key, v = key[order], v[order]
    if key.size:
        first = np.ones(key.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        vals = np.zeros(int(first.sum()))
        np.add.at(vals, np.cumsum(first) - 1, v)
        key = key[first]
    else:
        vals = v
    cc = key // max(rows, 1)
    ptr = np.zeros(cols + 1, _I)
    np.cumsum(np.bincount(cc, minlength=cols), out=ptr[1:])
    return SparseMatrixCSC(rows, cols, ptr, key - cc * max(rows, 1), vals)


def as_csc(M, rows: int, cols: int) -> SparseMatrixCSC:
    """Matrix-like -> CSC (reference: api.py:20-45).

    Accepts SparseMatrixCSC, the reference package's own CSC dataclass (duck
    typed), scipy sparse (any format), a dense 2-D array, or None.
    """
    if M is None:
        return empty_csc(rows, cols)
    if isinstance(M, SparseMatrixCSC):
        return M
    if all(hasattr(M, a) for a in ("col_pointers", "row_indices", "values")):
        return SparseMatrixCSC(rows, cols, np.asarray(M.col_pointers, _I),
                               np.asarray(M.row_indices, _I), np.asarray(M.values, _F))
    if hasattr(M, "tocsc") and not hasattr(M, "indptr"):
        M = M.tocsc()
    if hasattr(M, "indptr"):
        if hasattr(M, "format") and M.format != "csc":
            M = M.tocsc()
        if hasattr(M, "sort_indices"):
            M.sort_indices()
        return SparseMatrixCSC(rows, cols, np.asarray(M.indptr, _I),
                               np.asarray(M.indices, _I), np.asarray(M.data, _F))
    dense = np.asarray(M, dtype=_F)
    if dense.ndim != 2:
        raise TypeError("expected a matrix-like object")
    r, c = np.nonzero(dense)
    return csc_from_triplets(rows, cols, (r, c, dense[r, c]))
