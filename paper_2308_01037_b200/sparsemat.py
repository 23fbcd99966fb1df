"""Host-side sparse matrix type of the drop-in (reference sparsemat.py:29-146).

Holds the same (row, col, value) triples in CSR and CSC form (scipy arrays),
plus the provenance fields of the reference type.  Anything exposing
``.csr``/``.csc`` scipy arrays -- including the reference's own
``SparseMatrix`` -- is accepted by the estimators, so this type only exists so
the package runs where the reference is not installed.  File parsers, the
cleanup filters and digraph symmetrisation are in ingest.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy import sparse

from .errors import ArgumentError


@dataclass
class SparseMatrix:
    csr: sparse.csr_array
    csc: sparse.csc_array
    symmetric_hint: bool = False
    original_ids: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.csr.shape[0]

    @property
    def nnz(self) -> int:
        return self.csr.nnz

    @classmethod
    def from_coo(cls, rows, cols, vals, n: int, symmetric_hint: bool = False, original_ids=None, meta=None):
        """Triples -> matrix; duplicates, explicit zeros and out-of-range ids are
        rejected (reference sparsemat.py:61-100 contract)."""
        r = np.asarray(rows, dtype=np.int64)
        c = np.asarray(cols, dtype=np.int64)
        v = np.asarray(vals, dtype=np.float64)
        if not (r.shape == c.shape == v.shape):
            raise ArgumentError("rows, cols and vals must have equal length")
        if n <= 0:
            raise ArgumentError("matrix dimension must be positive")
        if r.size:
            if min(r.min(), c.min()) < 0 or max(r.max(), c.max()) >= n:
                raise ArgumentError(f"indices out of range for n={n}")
            if (v == 0.0).any():
                raise ArgumentError("explicit zero values are not stored")
            flat = r * np.int64(n) + c
            if np.unique(flat).size != flat.size:
                raise ArgumentError("duplicate (row, col) entries")
        m = sparse.coo_array((v, (r, c)), shape=(n, n))
        a_csr = m.tocsr()
        a_csr.sort_indices()
        a_csc = m.tocsc()
        a_csc.sort_indices()
        ids = None if original_ids is None else np.asarray(original_ids, dtype=np.int64)
        return cls(a_csr, a_csc, symmetric_hint, ids, dict(meta or {}))

    @classmethod
    def from_csr_arrays(cls, n, row_ptr, col_ids, vals, symmetric_hint=False, meta=None):
        """Wrap already sorted, duplicate-free CSR arrays without copying them
        (generators use this; pinned host buffers stay pinned)."""
        rp = np.asarray(row_ptr)
        ci = np.asarray(col_ids)
        va = np.asarray(vals, dtype=np.float64)
        a_csr = sparse.csr_array((n, n))
        a_csr.indptr, a_csr.indices, a_csr.data = rp, ci, va
        a_csr.has_sorted_indices = True
        if symmetric_hint:  # A == A^T: the CSC view shares the CSR arrays
            a_csc = sparse.csc_array((n, n))
            a_csc.indptr, a_csc.indices, a_csc.data = rp, ci, va
            a_csc.has_sorted_indices = True
        else:
            a_csc = a_csr.tocsc()
            a_csc.sort_indices()
        return cls(a_csr, a_csc, symmetric_hint, None, dict(meta or {}))

    @classmethod
    def from_dense(cls, arr, symmetric_hint: bool = False):
        d = np.asarray(arr, dtype=np.float64)
        if d.ndim != 2 or d.shape[0] != d.shape[1]:
            raise ArgumentError("dense input must be a square 2-D array")
        r, c = np.nonzero(d)
        return cls.from_coo(r, c, d[r, c], d.shape[0], symmetric_hint)

    def row_entries(self, i: int):
        lo, hi = self.csr.indptr[i], self.csr.indptr[i + 1]
        return self.csr.indices[lo:hi], self.csr.data[lo:hi]

    def col_entries(self, j: int):
        lo, hi = self.csc.indptr[j], self.csc.indptr[j + 1]
        return self.csc.indices[lo:hi], self.csc.data[lo:hi]

    def diagonal(self) -> np.ndarray:
        return self.csr.diagonal()

    def toarray(self) -> np.ndarray:
        return self.csr.toarray()


def scale(a, gamma: float):
    """Every stored value times gamma > 0 (reference sparsemat.py:338-352)."""
    if not gamma > 0:
        raise ArgumentError(f"gamma must be positive, got {gamma}")
    meta = dict(getattr(a, "meta", {}) or {})
    meta["gamma"] = meta.get("gamma", 1.0) * gamma
    a_csr = sparse.csr_array(a.csr * gamma)
    a_csc = sparse.csc_array(a.csc * gamma)
    return SparseMatrix(a_csr, a_csc, getattr(a, "symmetric_hint", False), getattr(a, "original_ids", None), meta)


def row_abs_sums(a) -> np.ndarray:
    """Per-row sum of |a_ij| (sequential, CSR order; zero for empty rows)."""
    out = np.zeros(a.csr.shape[0])
    if a.csr.nnz:
        rows = np.repeat(np.arange(a.csr.shape[0]), np.diff(a.csr.indptr))
        np.add.at(out, rows, np.abs(a.csr.data))
    return out
