"""Graph ingest: load_graph for edge lists and coordinate
Matrix Market files, the cleanup filters, and the Eq. 25 bipartite
symmetrization -- the reference's sparsemat.py:149-335 with the same names,
arguments, filter order, id compaction and errors.

Parsing is host text work (C++ in libmcfunm_gen.so, one pass).  The filters
are sort/unique/scatter over the edge arrays and run with torch on the device
(``device``; the GPU by default): drop loops, expand undirected edges, sort +
unique the (u, v) keys, compact ids of isolated nodes, and build the CSR.
The result is this package's SparseMatrix (host CSR/CSC, values 1), equal to
the reference's for the same file.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
from scipy import sparse

from .errors import ArgumentError, DataError, DegenerateInputError, ParseError
from .sparsemat import SparseMatrix

_GEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmcfunm_gen.so")


@dataclass
class GraphSource:
    """A graph file plus the cleanup filters to apply (sparsemat.py:149-163).

    format : "edgelist" or "matrix-market" ("mtx")
    directed : if False, every edge (u, v) also stores (v, u)
    """

    path: str | Path
    format: str = "edgelist"
    directed: bool = False
    drop_loops: bool = True
    drop_duplicates: bool = True
    drop_isolated: bool = True


_MESSAGES = {
    1: "expected at least two columns",
    2: "node ids must be integers",
    3: "node ids must be non-negative",
    10: "missing MatrixMarket header",
    11: "only 'matrix coordinate' files are supported",
    12: "unsupported value type",
    13: "unsupported storage",
    14: "size line must be 'rows cols nnz'",
    15: "adjacency matrix must be square",
    17: "malformed entry",
    18: "index out of declared range",
}


def _lib():
    lib = C.CDLL(_GEN)
    lib.mcfgen_parse_open.restype = C.c_void_p
    lib.mcfgen_parse_open.argtypes = [C.c_char_p, C.c_int]
    lib.mcfgen_parsed_info.restype = C.c_int64
    lib.mcfgen_parsed_info.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int)]
    lib.mcfgen_parsed_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.mcfgen_parse_close.argtypes = [C.c_void_p]
    return lib


def parse_edges(path, fmt: str):
    """(u, v) int64 edge arrays of an edge list (sparsemat.py:165-184) or a
    coordinate Matrix Market file (:187-245, symmetric storage expanded,
    zero values skipped, 0-based ids)."""
    path = Path(path)
    lib = _lib()
    h = lib.mcfgen_parse_open(str(path).encode(), 0 if fmt == "edgelist" else 1)
    try:
        err, line, cols = C.c_int(), C.c_int64(), C.c_int()
        m = lib.mcfgen_parsed_info(h, C.byref(err), C.byref(line), C.byref(cols))
        if m < 0:
            if err.value == 4:
                raise DataError(f"input file not found: {path}")
            if err.value == 16:
                raise ParseError(f"{path}:{line.value}: expected {cols.value} columns")
            if err.value == 19:
                raise ParseError(f"{path}: missing size line")
            raise ParseError(f"{path}:{line.value}: {_MESSAGES.get(err.value, 'parse error')}")
        u = np.empty(m, dtype=np.int64)
        v = np.empty(m, dtype=np.int64)
        if m:
            lib.mcfgen_parsed_copy(h, u.ctypes.data, v.ctypes.data)
        return u, v
    finally:
        lib.mcfgen_parse_close(h)


def _device(device):
    import torch
    if device is not None:
        return torch.device(device)
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def simple_graph_from_edges(u, v, directed: bool = False, drop_loops: bool = True, drop_duplicates: bool = True,
                            drop_isolated: bool = True, meta=None, device=None) -> SparseMatrix:
    """Filters in the reference's order (sparsemat.py:248-298): loops,
    undirected expansion, duplicate removal, isolated-node removal with id
    compaction; all stored values 1.  The sort/unique/remap run with torch on
    ``device``."""
    import torch
    dev = _device(device)
    u = torch.as_tensor(np.asarray(u, dtype=np.int64)).to(dev)
    v = torch.as_tensor(np.asarray(v, dtype=np.int64)).to(dev)
    if dev.type == "cuda":
        return _simple_graph_kernels(u, v, directed, drop_loops, drop_duplicates, drop_isolated, meta)
    if drop_loops and u.numel():
        keep = u != v
        u, v = u[keep], v[keep]
    if not directed and u.numel():
        u, v = torch.cat([u, v]), torch.cat([v, u])
    if u.numel() == 0:
        raise DegenerateInputError("graph is empty after filtering")
    top = int(torch.maximum(u.max(), v.max()).item()) + 1
    shift = max(1, int(top - 1).bit_length())
    if 2 * shift > 62:
        raise ArgumentError("node ids too large for 64-bit edge keys")
    key = (u << shift) | v
    if drop_duplicates:
        key = torch.unique(key, sorted=True)
    else:
        key = torch.sort(key).values
        if key.numel() > 1 and bool((key[1:] == key[:-1]).any()):
            raise ArgumentError("duplicate (row, col) entries")  # the reference's SparseMatrix.from_coo check
    u, v = key >> shift, key & ((1 << shift) - 1)
    original_ids = None
    if drop_isolated:
        present = torch.unique(torch.cat([u, v]), sorted=True)
        n = int(present.numel())
        if n != int(present[-1].item()) + 1:
            u = torch.searchsorted(present, u)
            v = torch.searchsorted(present, v)
            original_ids = present.cpu().numpy()
    else:
        n = top
    # keys are sorted by (u, v): the CSR rows come out in order, columns sorted
    counts = torch.bincount(u, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    csr = sparse.csr_array((np.ones(int(u.numel())), v.cpu().numpy(), row_ptr.cpu().numpy()), shape=(n, n))
    csr.has_sorted_indices = True
    csc = sparse.csc_array(csr.tocsc())
    csc.sort_indices()
    return SparseMatrix(csr, csc, not directed, original_ids, dict(meta or {}))


def _simple_graph_kernels(u, v, directed, drop_loops, drop_duplicates, drop_isolated, meta) -> SparseMatrix:
    """The same filters as library kernels (mcf_edges_to_csr: loops, undirected
    expansion, duplicates, sorted rows; mcf_csr_compact: isolated nodes)."""
    import torch

    from . import _native as N
    from .graphs import compact_isolated_device, edges_to_csr_device
    if u.numel() == 0:
        raise DegenerateInputError("graph is empty after filtering")
    top = int(torch.maximum(u.max(), v.max()).item()) + 1
    if top >= (1 << 31) or int(torch.minimum(u.min(), v.min()).item()) < 0:
        raise ArgumentError("node ids must lie in [0, 2^31)")
    keys = (u << 32) | v
    flags = ((N.MCF_EDGES_DROP_LOOPS if drop_loops else 0) | (0 if directed else N.MCF_EDGES_ADD_REVERSE)
             | (0 if drop_duplicates else N.MCF_EDGES_FAIL_ON_DUPLICATES))
    row_ptr, col_ids = edges_to_csr_device(keys, top, flags)
    if col_ids.numel() == 0:
        raise DegenerateInputError("graph is empty after filtering")
    n, original_ids = top, None
    if drop_isolated:
        k, row_ptr, col_ids, old = compact_isolated_device(top, row_ptr, col_ids)
        if k != top:
            n, original_ids = k, old.cpu().numpy()
    csr = sparse.csr_array((np.ones(int(col_ids.numel())), col_ids.cpu().numpy(), row_ptr.cpu().numpy()), shape=(n, n))
    csr.has_sorted_indices = True
    csc = sparse.csc_array(csr.tocsc())
    csc.sort_indices()
    return SparseMatrix(csr, csc, not directed, original_ids, dict(meta or {}))


def load_graph(source: GraphSource, device=None) -> SparseMatrix:
    """Read a graph file; return its binary adjacency matrix with the
    requested filters applied (sparsemat.py:301-317)."""
    path = Path(source.path)
    if not path.exists():
        raise DataError(f"input file not found: {path}")
    if source.format == "edgelist":
        u, v = parse_edges(path, "edgelist")
    elif source.format in ("matrix-market", "mtx"):
        u, v = parse_edges(path, "matrix-market")
    else:
        raise ArgumentError(f"unknown graph format '{source.format}'")
    return simple_graph_from_edges(u, v, directed=source.directed, drop_loops=source.drop_loops,
                                   drop_duplicates=source.drop_duplicates, drop_isolated=source.drop_isolated,
                                   meta={"source": str(path), "format": source.format, "directed": source.directed},
                                   device=device)


def symmetrize_digraph(a) -> SparseMatrix:
    """Bipartite symmetrization (Eq. 25, sparsemat.py:320-335): the 2n x 2n
    block matrix [[0, A], [A^T, 0]] -- out-copies are rows 0..n-1, in-copies
    n..2n-1."""
    csr = sparse.csr_array(a.csr)
    n = int(csr.shape[0])
    block = None
    if csr.nnz and np.all(csr.data == 1.0):
        import torch
        if torch.cuda.is_available():  # binary adjacency: the block structure built by the library kernels
            from .graphs import edges_to_csr_device
            coo = csr.tocoo()
            i = torch.from_numpy(coo.row.astype(np.int64)).cuda()
            j = torch.from_numpy(coo.col.astype(np.int64)).cuda() + n
            keys = torch.cat([(i << 32) | j, (j << 32) | i])  # (i, n + j) and its transpose (n + j, i)
            rp, ci = edges_to_csr_device(keys, 2 * n, 0)
            block = sparse.csr_array((np.ones(int(ci.numel())), ci.cpu().numpy(), rp.cpu().numpy()),
                                     shape=(2 * n, 2 * n))
            block.has_sorted_indices = True
    if block is None:
        block = sparse.csr_array(sparse.bmat([[None, csr], [csr.T, None]], format="csr"))
        block.sort_indices()
    meta = dict(getattr(a, "meta", None) or {})
    meta["symmetrized_blocks"] = int(csr.shape[0])
    if getattr(a, "original_ids", None) is not None:
        meta["source_original_ids"] = list(np.asarray(a.original_ids).tolist())
    csc = sparse.csc_array(block.tocsc())
    csc.sort_indices()
    return SparseMatrix(block, csc, True, None, meta)
