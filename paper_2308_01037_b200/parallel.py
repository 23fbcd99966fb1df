"""Multi-GPU execution: one process per GPU, graph replicated, start columns
sharded.

Every column's walks run on exactly one rank; the Philox stream is keyed by
(seed, column, walk, step), so a column produces the same bits wherever it
runs.  The only exchange is assembling the per-column results:
  * action: q (8 n bytes) -- each rank contributes its own column range, the
    rest of its vector is zero, so a SUM all-reduce is an exact concatenation;
    then y over the rank's row range, assembled the same way;
  * diag: the per-entry partials pcol (8 nnz bytes), assembled the same way,
    then d over the rank's row range.
Results are therefore bitwise identical for 1, 2, 4 and 8 GPUs.

sharded_action_peer folds the action exchange into the combine instead: the
ranks map each other's q and y buffers (CUDA IPC over NVLink) and one SpMV per
rank gathers q from the owning ranks and writes its y rows into every rank's
buffer (mcf_spmv_peer) -- two barriers, no NCCL on the data path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .device import DeviceGraph, WalkParams
from .series import as_stream
from .walker import check_config


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def column_shards(walk_pre, parts: int):
    """Contiguous column ranges with ~equal walk counts (walk_pre: n+1 prefix)."""
    if torch.is_tensor(walk_pre):  # search on the device, copy back parts+1 ints
        n = walk_pre.numel() - 1
        k = torch.arange(1, parts, device=walk_pre.device, dtype=torch.int64)
        tgt = (walk_pre[-1] * k + parts - 1) // parts
        inner = torch.searchsorted(walk_pre, tgt, side="left").cpu().numpy()
    else:
        pre = np.asarray(walk_pre, dtype=np.int64)
        n = pre.size - 1
        tgt = (int(pre[-1]) * np.arange(1, parts) + parts - 1) // parts
        inner = np.searchsorted(pre, tgt, side="left")
    cuts = np.concatenate([[0], inner, [n]])
    cuts = np.maximum.accumulate(np.minimum(cuts, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def _shards(peers, g, pre, n_walks: int, parts: int):
    """column_shards, remembered per (graph, N_s, parts) on the peer buffers."""
    key = (id(g), int(n_walks), int(parts))
    hit = peers.shard_cache.get(key)
    if hit is None or hit[0] is not g:
        hit = (g, column_shards(pre, parts))
        peers.shard_cache[key] = hit
    return hit[1]


def row_shards(n: int, parts: int):
    b = [n * k // parts for k in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts)]


def assemble(t: torch.Tensor, group=None) -> torch.Tensor:
    """Disjoint per-rank pieces (zeros elsewhere) -> full vector on every rank."""
    if world()[1] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (zero-copy torch view)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (int(ptr), False), "version": 3}


def _device_view(ptr: int, n: int, device) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, n), device=device)


class _Raw:
    """A raw device pointer where the binding expects a tensor (data_ptr())."""

    def __init__(self, ptr: int):
        self.ptr = int(ptr)

    def data_ptr(self) -> int:
        return self.ptr


class PeerBuffers:
    """Per-rank device buffers every rank of the node can read and write over
    NVLink: each rank allocates its own (mcf_peer_alloc), the 64-byte CUDA IPC
    handles are swapped with an all-gather over ``group``, and every rank maps
    the others' (mcf_peer_open).  ptrs[k][b] is buffer b of rank k as seen by
    this process (its own are local)."""

    def __init__(self, nbytes: list[int], group=None):
        rank, size = world()
        self.rank = rank
        # column shards by (graph, N_s, ranks): a function of the budgets only,
        # so repeated passes skip the device-to-host read that finds them
        self.shard_cache = {}
        self.own, handles = [], []
        for b in nbytes:
            ptr, h = C.c_void_p(), C.create_string_buffer(64)
            N.check(N.lib().mcf_peer_alloc(int(b), C.byref(ptr), h), "mcf_peer_alloc")
            self.own.append(ptr.value)
            handles.append(h.raw)
        allh = [None] * size
        dist.all_gather_object(allh, handles, group=group)
        self.ptrs, self.opened = [], []
        for k in range(size):
            if k == rank:
                self.ptrs.append(list(self.own))
                continue
            row = []
            for h in allh[k]:
                ptr = C.c_void_p()
                N.check(N.lib().mcf_peer_open(C.create_string_buffer(h, 64), C.byref(ptr)), "mcf_peer_open")
                row.append(ptr.value)
                self.opened.append(ptr.value)
            self.ptrs.append(row)

    def close(self, group=None):
        torch.cuda.synchronize()
        dist.barrier(group=group)  # nobody still reads our buffers
        for p in self.opened:
            N.lib().mcf_peer_close(C.c_void_p(p))
        dist.barrier(group=group)
        for p in self.own:
            N.lib().mcf_peer_free(C.c_void_p(p))
        self.opened, self.own = [], []


def sharded_action_peer(g: DeviceGraph, coeffs, v, config, *, params=None, group=None, peers: PeerBuffers = None):
    """Multi-GPU RandFunmAction with the exchange folded into the combine:
    each rank walks its column shard into its own q buffer; after a barrier
    one SpMV per rank gathers q[j] from the rank owning column j (peer memory
    over NVLink) and writes its row shard of y into every rank's y buffer
    (mcf_spmv_peer) -- no all-gather of q or y.  ``v=None`` is v = 1.
    Returns (y, stats); y holds all rows on every rank."""
    rank, size = world()
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    z = coeffs.prefix(cfg.max_steps + 2)
    params = params or WalkParams(cfg, z, g.device)
    if v is None:
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
    own = peers is None
    if own:
        peers = PeerBuffers([8 * g.n, 8 * g.n], group)
    ni, pre = g.allocate(cfg.n_walks)
    shards = _shards(peers, g, pre, cfg.n_walks, size)
    bounds = [shards[0][0]] + [b for _, b in shards]
    st = g.new_stats()
    r = g.spmv(v)
    g.walk_action(params, pre, r, _Raw(peers.ptrs[rank][0]), cols=shards[rank], stats=st)
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank's q shard is complete
    g.spmv_peer([peers.ptrs[k][0] for k in range(size)], bounds, [peers.ptrs[k][1] for k in range(size)],
                alpha=z[0], v=v, beta=z[1], r=r, rows=row_shards(g.n, size)[rank])
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank's y rows have landed everywhere
    y = _device_view(peers.ptrs[rank][1], g.n, g.device).clone()
    if own:
        peers.close(group)
    return y, st


def sharded_diag_peer(g: DeviceGraph, coeffs, config, *, params=None, group=None, peers: PeerBuffers = None):
    """Multi-GPU RandFunmDiag with the exchange folded into the combine: each
    rank writes the Eq. 20 partials of its column shard into its own pcol
    buffer; after a barrier one kernel per rank reads every pcol[(i, c)] from
    the rank owning column c (peer memory) and writes its rows of d into every
    rank's d buffer (mcf_diag_combine_peer).  Returns (d, stats)."""
    rank, size = world()
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    z = coeffs.prefix(cfg.max_steps + 2)
    params = params or WalkParams(cfg, z, g.device)
    own = peers is None
    if own:
        peers = PeerBuffers([8 * g.nnz, 8 * g.n], group)
    ni, pre = g.allocate(cfg.n_walks)
    shards = _shards(peers, g, pre, cfg.n_walks, size)
    bounds = [shards[0][0]] + [b for _, b in shards]
    st = g.new_stats()
    _device_view(peers.ptrs[rank][0], g.nnz, g.device).zero_()  # columns without walks keep zero partials
    g.walk_diag(params, pre, _Raw(peers.ptrs[rank][0]), cols=shards[rank], stats=st)
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank's partials are complete
    g.diag_combine_peer(z[0], z[1], [peers.ptrs[k][0] for k in range(size)], bounds,
                        [peers.ptrs[k][1] for k in range(size)], rows=row_shards(g.n, size)[rank])
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank's d rows have landed everywhere
    d = _device_view(peers.ptrs[rank][1], g.n, g.device).clone()
    if own:
        peers.close(group)
    return d, st


def sharded_action(g: DeviceGraph, coeffs, v, config, *, params=None, budgets=None, group=None):
    """One RandFunmAction pass with this rank's share of the start columns.
    ``v=None`` is v = 1.  Returns (y, stats) with y assembled on every rank."""
    rank, size = world()
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    z = coeffs.prefix(cfg.max_steps + 2)
    params = params or WalkParams(cfg, z, g.device)
    if size == 1 and budgets is None:  # the whole pass in one library call (q, y, stats overwritten)
        q = torch.empty(g.n, dtype=torch.float64, device=g.device)
        r, y = torch.empty_like(q), torch.empty_like(q)
        st = torch.empty(N.MCF_STATS_LEN, dtype=torch.int64, device=g.device)
        return g.funm_action(params, cfg.n_walks, v, z[0], z[1], r, q, y, stats=st, want_ni=False)[0], st
    if v is None:
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
    ni, pre = budgets if budgets is not None else g.allocate(cfg.n_walks)
    st = g.new_stats()
    cols = column_shards(pre, size)[rank]
    rows = row_shards(g.n, size)[rank]
    r = g.spmv(v)
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    g.walk_action(params, pre, r, q, cols=cols, stats=st)
    assemble(q, group)
    y = torch.zeros(g.n, dtype=torch.float64, device=g.device) if size > 1 else None
    y = g.spmv(q, alpha=z[0], v=v, beta=z[1], r=r, out=y, rows=rows)
    assemble(y, group)
    return y, st


def sharded_diag(g: DeviceGraph, coeffs, config, *, params=None, budgets=None, group=None):
    """One RandFunmDiag pass with this rank's share of the start columns."""
    rank, size = world()
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    z = coeffs.prefix(cfg.max_steps + 2)
    params = params or WalkParams(cfg, z, g.device)
    ni, pre = budgets if budgets is not None else g.allocate(cfg.n_walks)
    st = g.new_stats()
    cols = column_shards(pre, size)[rank] if size > 1 else (0, g.n)
    rows = row_shards(g.n, size)[rank] if size > 1 else (0, g.n)
    pcol = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    g.walk_diag(params, pre, pcol, cols=cols, stats=st)
    assemble(pcol, group)
    d = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    g.diag_combine(z[0], z[1], pcol, d, rows=rows)
    assemble(d, group)
    return d, st
