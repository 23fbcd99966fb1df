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
"""

from __future__ import annotations

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


def row_shards(n: int, parts: int):
    b = [n * k // parts for k in range(parts + 1)]
    return [(b[i], b[i + 1]) for i in range(parts)]


def assemble(t: torch.Tensor, group=None) -> torch.Tensor:
    """Disjoint per-rank pieces (zeros elsewhere) -> full vector on every rank."""
    if world()[1] > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


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
