"""Synthetic benchmark graphs for the BASELINE.json configs (workload
generation, not the hot path).  All return this package's SparseMatrix with
symmetric 0/1 values; callers scale by beta = 1 / lambda_max."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
from scipy import sparse

from .errors import ArgumentError
from .sparsemat import SparseMatrix

_GEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libmcfunm_gen.so")


def _gen_lib():
    lib = C.CDLL(_GEN)
    lib.mcfgen_ba_nnz.restype = C.c_int64
    lib.mcfgen_ba_nnz.argtypes = [C.c_int64, C.c_int64]
    lib.mcfgen_barabasi_albert.restype = C.c_int64
    lib.mcfgen_barabasi_albert.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p]
    return lib


def _alloc(shape, dtype, pinned):
    if pinned:
        import torch
        t = torch.empty(shape, dtype={np.int64: torch.int64, np.int32: torch.int32,
                                      np.float64: torch.float64}[dtype], pin_memory=True)
        return t.numpy()
    return np.empty(shape, dtype=dtype)


def barabasi_albert(n: int, m: int, seed: int = 0, pinned: bool = False) -> SparseMatrix:
    """BASELINE config 2 graph (n = 1e6, m = 4 -> nnz 7,999,968)."""
    lib = _gen_lib()
    nnz = lib.mcfgen_ba_nnz(n, m)
    if nnz < 0:
        raise ArgumentError("need m >= 1 and n > m + 1")
    rp = _alloc(n + 1, np.int64, pinned)
    ci = _alloc(nnz, np.int32, pinned)
    got = lib.mcfgen_barabasi_albert(n, m, seed, rp.ctypes.data, ci.ctypes.data)
    assert got == nnz
    vals = _alloc(nnz, np.float64, pinned)
    vals[:] = 1.0
    meta = {"generator": "barabasi-albert", "n": n, "m": m, "seed": seed, "nnz": int(nnz)}
    return SparseMatrix.from_csr_arrays(n, rp, ci, vals, symmetric_hint=True, meta=meta)


def erdos_renyi_lcc(n: int, mean_degree: float, seed: int = 0) -> SparseMatrix:
    """BASELINE config 1 graph: G(n, m = n d / 2 random pairs), simple,
    undirected, largest connected component only (ids compacted)."""
    from scipy.sparse.csgraph import connected_components
    rng = np.random.default_rng(seed)
    m = int(n * mean_degree / 2)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    keep = u != v
    u, v = u[keep], v[keep]
    a = sparse.coo_array((np.ones(2 * u.size), (np.r_[u, v], np.r_[v, u])), shape=(n, n)).tocsr()
    a.sum_duplicates()
    a.data[:] = 1.0
    _, lab = connected_components(a, directed=False)
    big = np.flatnonzero(lab == np.argmax(np.bincount(lab)))
    sub = sparse.csr_array(a[big][:, big])
    sub.sort_indices()
    out = SparseMatrix.from_csr_arrays(big.size, sub.indptr.astype(np.int64), sub.indices.astype(np.int32),
                                       sub.data, symmetric_hint=True,
                                       meta={"generator": "erdos-renyi-lcc", "n0": n, "seed": seed})
    out.original_ids = big
    return out


def lambda_max(a) -> float:
    """Largest eigenvalue of a symmetric matrix (ARPACK, deterministic start
    vector, so every process computes the same fp64 beta)."""
    from scipy.sparse.linalg import eigsh
    m = sparse.csr_array(a.csr, dtype=np.float64)
    if m.shape[0] <= 512:
        return float(np.linalg.eigvalsh(m.toarray())[-1])
    return float(eigsh(m, k=1, which="LA", v0=np.ones(m.shape[0]), tol=1e-12)[0][0])


# --------------------------------------------------------------------------
# device generators (large configs; torch is plumbing here, the estimator
# kernels never see these code paths)
# --------------------------------------------------------------------------
def _csr_from_sorted_keys(keys, scale: int, n: int):
    import torch
    rows = keys >> scale
    cols = (keys & (n - 1)).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=keys.device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    return row_ptr, cols


def rmat_torch(scale: int, edge_factor: int = 16, pa: float = 0.57, pb: float = 0.19, pc: float = 0.19,
                seed: int = 0, device="cuda", chunk: int = 1 << 26):
    """Symmetrised R-MAT with torch ops (the bench recipe, tools/bench_graphs.py,
    which must load no repository library): edge_factor * 2^scale
    draws, one uniform per level with the reference's quadrant rule
    (graphgen.py:138-143: row bit r >= pa+pb, column bit r in [pa, pa+pb) or
    r >= pa+pb+pc), then both directions, loops and duplicates removed.  No
    isolated-node compaction: n = 2^scale rows as generated.
    Returns (n, row_ptr int64, col_ids int32) on the device."""
    import torch
    n = 1 << scale
    draws = edge_factor << scale
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    ab, abc = pa + pb, pa + pb + pc
    keys = []
    for lo in range(0, draws, chunk):
        m = min(chunk, draws - lo)
        u = torch.zeros(m, dtype=torch.int64, device=device)
        v = torch.zeros(m, dtype=torch.int64, device=device)
        for _ in range(scale):
            r = torch.rand(m, generator=gen, dtype=torch.float64, device=device)
            rb = r >= ab
            cb = ((r >= pa) & ~rb) | (r >= abc)
            u = (u << 1) | rb
            v = (v << 1) | cb
        keep = u != v
        u, v = u[keep], v[keep]
        keys.append((u << scale) | v)
        keys.append((v << scale) | u)
    k = torch.cat(keys)
    del keys
    k = torch.unique(k, sorted=True)
    row_ptr, cols = _csr_from_sorted_keys(k, scale, n)
    return n, row_ptr, cols


def edges_to_csr_device(keys, n: int, flags: int):
    """Edge keys (u << 32) | v (int64 tensor on the GPU) -> CSR (row_ptr int64,
    col_ids int32) with the library's cleanup kernels (mcf_edges_to_csr)."""
    import ctypes as C

    import torch

    from . import _native as N
    dev = keys.device
    cap = keys.numel() * (2 if flags & N.MCF_EDGES_ADD_REVERSE else 1)
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col_ids = torch.empty(max(1, cap), dtype=torch.int32, device=dev)
    nnz = C.c_int64()
    s = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib().mcf_edges_to_csr(keys.data_ptr(), keys.numel(), int(n), int(flags), row_ptr.data_ptr(),
                                     col_ids.data_ptr(), int(cap), C.byref(nnz), s), "mcf_edges_to_csr")
    return row_ptr, col_ids[:nnz.value]


def compact_isolated_device(n: int, row_ptr, col_ids):
    """Drop the nodes with no incident edge, renumbering the rest in order
    (mcf_csr_compact).  Returns (n_out, row_ptr, col_ids, original_ids)."""
    import ctypes as C

    import torch

    from . import _native as N
    dev = row_ptr.device
    new_rp = torch.empty(n + 1, dtype=torch.int64, device=dev)
    old = torch.empty(n, dtype=torch.int64, device=dev)
    n_out = C.c_int64()
    s = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib().mcf_csr_compact(int(n), row_ptr.data_ptr(), col_ids.data_ptr(), col_ids.numel(),
                                    new_rp.data_ptr(), old.data_ptr(), C.byref(n_out), s), "mcf_csr_compact")
    k = n_out.value
    return k, new_rp[:k + 1].clone(), col_ids, old[:k].clone()


def rmat_device(scale: int, edge_factor: int = 16, pa: float = 0.57, pb: float = 0.19, pc: float = 0.19,
                seed: int = 0, device="cuda"):
    """Symmetrised R-MAT generated by the library kernels (mcf_gen_rmat_keys:
    edge_factor * 2^scale draws of the reference's quadrant rule,
    graphgen.py:138-143; mcf_edges_to_csr: loops dropped, both directions,
    duplicates merged, rows sorted).  No isolated-node compaction: n = 2^scale
    rows.  Returns (n, row_ptr int64, col_ids int32) on the device."""
    import torch

    from . import _native as N
    n = 1 << scale
    draws = edge_factor << scale
    keys = torch.empty(draws, dtype=torch.int64, device=device)
    s = torch.cuda.current_stream(keys.device).cuda_stream
    N.check(N.lib().mcf_gen_rmat_keys(int(scale), int(draws), float(pa), float(pb), float(pc),
                                      int(seed) & 0xFFFFFFFFFFFFFFFF, keys.data_ptr(), s), "mcf_gen_rmat_keys")
    row_ptr, col_ids = edges_to_csr_device(keys, n, N.MCF_EDGES_DROP_LOOPS | N.MCF_EDGES_ADD_REVERSE)
    return n, row_ptr, col_ids


def chung_lu_device(n: int, exponent: float = 2.1, mean_degree: float = 20.0, max_degree: float = 1e5,
                    seed: int = 0, device="cuda"):
    """Chung-Lu power-law graph by the library kernels: the truncated-Pareto
    expected degrees of chung_lu_torch, n mean / 2 edges whose endpoints are
    drawn from their cumulative distribution (mcf_gen_chung_lu_keys), then
    mcf_edges_to_csr.  Returns (n, row_ptr, col_ids) on the device."""
    import torch

    from . import _native as N
    a = exponent - 1.0

    def weights(wmin):
        u = (torch.arange(n, dtype=torch.float64, device=device) + 0.5) / n
        r = (wmin / max_degree) ** a
        return wmin * (1.0 - u * (1.0 - r)) ** (-1.0 / a)

    lo, hi = 1e-3, mean_degree
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if float(weights(mid).mean()) < mean_degree:
            lo = mid
        else:
            hi = mid
    w = torch.flip(weights(0.5 * (lo + hi)), [0])
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    m = int(round(n * mean_degree / 2))
    keys = torch.empty(m, dtype=torch.int64, device=device)
    s = torch.cuda.current_stream(keys.device).cuda_stream
    N.check(N.lib().mcf_gen_chung_lu_keys(cdf.data_ptr(), int(n), int(m), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                          keys.data_ptr(), s), "mcf_gen_chung_lu_keys")
    row_ptr, col_ids = edges_to_csr_device(keys, n, N.MCF_EDGES_DROP_LOOPS | N.MCF_EDGES_ADD_REVERSE)
    return n, row_ptr, col_ids


def lambda_max_device(g, iters: int = 300) -> float:
    """Largest eigenvalue of a symmetric nonnegative matrix on the device:
    power iteration on A + I (the +1 shift keeps -lambda_max away) with the
    library SpMV, Rayleigh quotient at the end."""
    import torch
    x = torch.ones(g.n, dtype=torch.float64, device=g.device)
    x /= torch.linalg.norm(x)
    y = torch.empty_like(x)
    for _ in range(iters):
        g.spmv(x, alpha=1.0, v=x, out=y)
        x, y = y / torch.linalg.norm(y), x
    g.spmv(x, out=y)
    return float((x @ y) / (x @ x))


def chung_lu_torch(n: int, exponent: float = 2.1, mean_degree: float = 20.0, max_degree: float = 1e5,
                    seed: int = 0, device="cuda", chunk: int = 1 << 26):
    """Chung-Lu power-law graph with torch ops (the bench recipe): expected
    degrees w_i from a truncated Pareto(exponent) on [w_min, max_degree] with
    w_min solved for the requested mean (deterministic quantiles, hubs first),
    n*mean/2 edges with both endpoints drawn proportionally to w, then both
    directions, loops and duplicates removed.  Returns (n, row_ptr, col_ids)."""
    import math

    import torch
    a = exponent - 1.0

    def weights(wmin):
        u = (torch.arange(n, dtype=torch.float64, device=device) + 0.5) / n
        r = (wmin / max_degree) ** a
        return wmin * (1.0 - u * (1.0 - r)) ** (-1.0 / a)

    lo, hi = 1e-3, mean_degree
    for _ in range(60):  # bisection on w_min for the mean degree
        mid = 0.5 * (lo + hi)
        if float(weights(mid).mean()) < mean_degree:
            lo = mid
        else:
            hi = mid
    w = torch.flip(weights(0.5 * (lo + hi)), [0])  # node 0 = largest expected degree
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    m = int(round(n * mean_degree / 2))
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    scale = int(math.ceil(math.log2(n)))
    keys = []
    for lo_ in range(0, m, chunk):
        k = min(chunk, m - lo_)
        u = torch.searchsorted(cdf, torch.rand(k, generator=gen, dtype=torch.float64, device=device)).clamp_(max=n - 1)
        v = torch.searchsorted(cdf, torch.rand(k, generator=gen, dtype=torch.float64, device=device)).clamp_(max=n - 1)
        keep = u != v
        u, v = u[keep], v[keep]
        keys.append((u << scale) | v)
        keys.append((v << scale) | u)
    kk = torch.unique(torch.cat(keys), sorted=True)
    del keys
    rows = kk >> scale
    cols = (kk & ((1 << scale) - 1)).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    return n, row_ptr, cols


def small_world(n: int, k: int, rewire_prob: float = 0.1, seed: int = 0) -> SparseMatrix:
    """Ring lattice (k/2 neighbours per side) with every lattice edge (i, j)
    rewired to (i, m), m uniform among non-neighbours of i, with probability
    rewire_prob (the paper's smallworld workload).  Host
    numpy generator for test-sized graphs."""
    if k % 2 or not 0 < k < n:
        raise ArgumentError("need an even k with 0 < k < n")
    rng = np.random.default_rng(seed)
    adj = [set() for _ in range(n)]
    for off in range(1, k // 2 + 1):
        for i in range(n):
            j = (i + off) % n
            adj[i].add(j)
            adj[j].add(i)
    for off in range(1, k // 2 + 1):
        for i in range(n):
            j = (i + off) % n
            if rng.random() >= rewire_prob or j not in adj[i] or len(adj[i]) >= n - 1:
                continue
            while True:
                m = int(rng.integers(n))
                if m != i and m not in adj[i]:
                    break
            adj[i].discard(j)
            adj[j].discard(i)
            adj[i].add(m)
            adj[m].add(i)
    rows = np.repeat(np.arange(n), [len(s) for s in adj])
    cols = np.concatenate([np.array(sorted(s), dtype=np.int64) for s in adj])
    return SparseMatrix.from_coo(rows, cols, np.ones(rows.size), n, symmetric_hint=True,
                                 meta={"generator": "smallworld", "n": n, "k": k, "p": rewire_prob, "seed": seed})
