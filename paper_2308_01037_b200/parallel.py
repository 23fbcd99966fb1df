"""Multi-GPU execution: one process per GPU, graph replicated, start columns
sharded.

Every column's walks run on exactly one rank; the Philox stream is keyed by
(seed, column, walk, step), so a column produces the same bits wherever it
runs.  Shards are contiguous column ranges balanced by a per-column cost
(``mcf_column_costs``: walks for action; emissions plus Eq. 20 combine probes
for diag -- the hub columns of R-MAT / Chung-Lu graphs hold most of the
combine work), and every call gets its shard's exact walk count as
walk_capacity (per-rank buffers are sized by the shard, not by N_s).  The
only exchange is assembling the per-column results:
  * action: q by column shard (all_gather_into_tensor of each rank's own
    range), then y by row shard;
  * diag: the per-entry partials of a column shard (a contiguous CSC range),
    then d by row shard.
Results are bitwise identical for 1, 2, 4 and 8 GPUs.

sharded_action_peer / sharded_diag_peer fold the exchange into the combine
instead: the ranks map each other's buffers (CUDA IPC over NVLink) and one
kernel per rank gathers q (or the partials) from the owning ranks and writes
its rows of y (or d) into every rank's buffer -- two barriers, no NCCL on the
data path.
"""

from __future__ import annotations

import ctypes as C
import weakref

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


def _cuts(prefix, parts: int):
    """Indices k_1..k_{parts-1} splitting a non-decreasing prefix (length n+1)
    into parts of ~equal total: k_j = first index with prefix >= j/parts of
    the total."""
    if torch.is_tensor(prefix):  # search on the device, copy back parts-1 ints
        k = torch.arange(1, parts, device=prefix.device, dtype=torch.int64)
        tgt = (prefix[-1] * k + parts - 1) // parts
        return torch.searchsorted(prefix, tgt, side="left").cpu().numpy()
    pre = np.asarray(prefix, dtype=np.int64)
    tgt = (int(pre[-1]) * np.arange(1, parts) + parts - 1) // parts
    return np.searchsorted(pre, tgt, side="left")


def column_shards(walk_pre, parts: int, cost=None):
    """Contiguous start-column ranges, one per rank.  Balanced by walk count
    (walk_pre: n+1 prefix), or -- with ``cost`` (per-column work, e.g.
    DeviceGraph.column_costs) -- by the prefix sum of the cost (SURVEY 8(e):
    "balanced by the prefix sum of N_i x expected length"; the paper fixes the
    same imbalance with dynamic scheduling)."""
    n = (walk_pre.numel() if torch.is_tensor(walk_pre) else len(walk_pre)) - 1
    if cost is None:
        inner = _cuts(walk_pre, parts)
    else:
        cp = torch.zeros(n + 1, dtype=torch.int64, device=cost.device) if torch.is_tensor(cost) else np.zeros(n + 1, np.int64)
        if torch.is_tensor(cost):
            torch.cumsum(cost, 0, out=cp[1:])
        else:
            cp[1:] = np.cumsum(np.asarray(cost, dtype=np.int64))
        inner = _cuts(cp, parts)
    cuts = np.concatenate([[0], inner, [n]])
    cuts = np.maximum.accumulate(np.minimum(cuts, n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def shard_walks(walk_pre, shards):
    """Walk count of every shard (the exact walk_capacity of its calls)."""
    idx = [shards[0][0]] + [b for _, b in shards]
    if torch.is_tensor(walk_pre):
        v = walk_pre[torch.tensor(idx, device=walk_pre.device)].cpu().numpy()
    else:
        v = np.asarray(walk_pre, dtype=np.int64)[idx]
    return [int(v[i + 1] - v[i]) for i in range(len(shards))]


def _shards(peers, g, pre, n_walks: int, parts: int, mode: str, max_steps: int):
    """Cost-balanced column shards and their walk counts, remembered per
    (graph, N_s, ranks, mode) on the peer buffers (a function of the budgets
    only, so repeated passes skip the device reads that find them)."""
    key = (id(g), int(n_walks), int(parts), mode, int(max_steps))
    hit = peers.shard_cache.get(key)
    if hit is None or hit[0]() is not g:
        cost = g.column_costs(pre, max_steps, mode) if parts > 1 else None
        sh = column_shards(pre, parts, cost)
        hit = (weakref.ref(g), sh, shard_walks(pre, sh))
        peers.shard_cache[key] = hit
    return hit[1], hit[2]


def row_shards(n: int, parts: int):
    b = [n * k // parts for k in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts)]


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
    ones = v is None
    if ones:
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
    own = peers is None
    if own:
        peers = PeerBuffers([8 * g.n, 8 * g.n], group)
    ni, pre = g.allocate(cfg.n_walks)
    shards, walks = _shards(peers, g, pre, cfg.n_walks, size, "action", cfg.max_steps)
    bounds = [shards[0][0]] + [b for _, b in shards]
    st = g.new_stats()
    r = g.spmv(None if ones else v)  # v = 1: CSR-order row sums, as the one-GPU mcf_funm_action
    g.walk_action(params.derive(capacity=walks[rank]), pre, r, _Raw(peers.ptrs[rank][0]), cols=shards[rank],
                  stats=st)
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
    shards, walks = _shards(peers, g, pre, cfg.n_walks, size, "diag", cfg.max_steps)
    bounds = [shards[0][0]] + [b for _, b in shards]
    st = g.new_stats()
    _device_view(peers.ptrs[rank][0], g.nnz, g.device).zero_()  # columns without walks keep zero partials
    g.walk_diag(params.derive(capacity=walks[rank]), pre, _Raw(peers.ptrs[rank][0]), cols=shards[rank], stats=st)
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


def gather_ranges(t: torch.Tensor, bounds, group=None) -> torch.Tensor:
    """Every rank holds its own slice t[bounds[r]:bounds[r+1]] (contiguous,
    disjoint, covering [bounds[0], bounds[-1])); after the call every rank
    holds all of them.  One NCCL all_gather_into_tensor of equal-length
    (padded) pieces: each rank sends only its own bytes, not a zero-padded
    full vector (an all-reduce moves twice as much)."""
    rank, size = world()
    if size == 1:
        return t
    lens = [int(bounds[k + 1] - bounds[k]) for k in range(size)]
    L = max(1, max(lens))
    # gloo (CPU tests, the shared-GPU functional mode) gathers host tensors
    dev = t.device if dist.get_backend(group) != "gloo" else torch.device("cpu")
    send = torch.zeros(L, dtype=t.dtype, device=dev)
    send[:lens[rank]] = t[bounds[rank]:bounds[rank + 1]].to(dev)
    recv = torch.empty(size * L, dtype=t.dtype, device=dev)
    dist.all_gather_into_tensor(recv, send, group=group)
    recv = recv.to(t.device)
    for k in range(size):
        if k != rank and lens[k]:
            t[bounds[k]:bounds[k + 1]] = recv[k * L:k * L + lens[k]]
    return t


def sharded_action(g: DeviceGraph, coeffs, v, config, *, params=None, budgets=None, group=None):
    """One RandFunmAction pass with this rank's share of the start columns.
    ``v=None`` is v = 1.  Returns (y, stats) with y assembled on every rank:
    q is all-gathered by column shard, y by row shard."""
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
    ones = v is None
    if ones:
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
    ni, pre = budgets if budgets is not None else g.allocate(cfg.n_walks)
    st = g.new_stats()
    shards = column_shards(pre, size)
    walks = shard_walks(pre, shards)
    rows = row_shards(g.n, size)
    r = g.spmv(None if ones else v)  # v = 1: CSR-order row sums, as the one-GPU mcf_funm_action
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    g.walk_action(params.derive(capacity=walks[rank]), pre, r, q, cols=shards[rank], stats=st)
    gather_ranges(q, [shards[0][0]] + [b for _, b in shards], group)
    y = torch.zeros(g.n, dtype=torch.float64, device=g.device) if size > 1 else None
    y = g.spmv(q, alpha=z[0], v=v, beta=z[1], r=r, out=y, rows=rows[rank])
    gather_ranges(y, [rows[0][0]] + [b for _, b in rows], group)
    return y, st


def sharded_diag(g: DeviceGraph, coeffs, config, *, params=None, budgets=None, group=None):
    """One RandFunmDiag pass with this rank's share of the start columns
    (cost-balanced shards).  The per-entry partials of a column shard are a
    contiguous CSC range, all-gathered; then d by row shard, all-gathered.
    Bitwise identical to one GPU."""
    rank, size = world()
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    z = coeffs.prefix(cfg.max_steps + 2)
    params = params or WalkParams(cfg, z, g.device)
    ni, pre = budgets if budgets is not None else g.allocate(cfg.n_walks)
    if size > 1:
        shards = column_shards(pre, size, g.column_costs(pre, cfg.max_steps, "diag"))
        walks = shard_walks(pre, shards)
        cols = shards[rank]
        cap = walks[rank]
    else:
        cols = (0, g.n)
        cap = int(pre[-1]) if budgets is not None else cfg.n_walks
    rows = row_shards(g.n, size)
    pcol = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    g.walk_diag(params.derive(capacity=cap), pre, pcol, cols=cols, stats=st)
    if size > 1:
        cb = g.csc_ptr[torch.tensor([shards[0][0]] + [b for _, b in shards], device=g.device)].cpu().numpy()
        gather_ranges(pcol, cb, group)
    d = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    g.diag_combine(z[0], z[1], pcol, d, rows=rows[rank])
    gather_ranges(d, [rows[0][0]] + [b for _, b in rows], group)
    return d, st
