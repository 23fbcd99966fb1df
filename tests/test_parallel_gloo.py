"""Multi-process host logic of the column-sharded path (parallel.py), world
size 2 over gloo on CPU.  The per-column compute is the oracle (test-only
stand-in for the device); what is under test is the cost-balanced sharding and
the exact assembly (all_gather of each rank's own range): sharded results must
equal the single-process result bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle import port
from paper_2308_01037_b200 import parallel
from tests import golden_io


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def column_costs_np(csc_ptr, csc_rows, row_ptr, ni, max_steps, mode="diag"):
    """numpy statement of mcf_column_costs (mcf_util.cu k_column_costs)."""
    n = len(ni)
    if mode == "action":
        return np.asarray(ni, dtype=np.int64).copy()
    deg = np.diff(row_ptr)
    m = np.asarray(ni, dtype=np.int64) * (max_steps + 1)
    col_of = np.repeat(np.arange(n), np.diff(csc_ptr))
    probes = np.minimum(deg[csc_rows], m[col_of])
    cost = np.zeros(n, dtype=np.int64)
    np.add.at(cost, col_of, probes)
    cost += 3 * m
    cost[np.asarray(ni) == 0] = 0
    return cost


def _per_entry_partials(c, t, z, ni, cols):
    """pcol[(i, c)] (CSC order) for the given columns, one oracle call per column."""
    a = c.sa
    pcol = np.zeros(a.csc_rows.size)
    for col in cols:
        contrib, _ = port.diag_columns(a, t, z, ni, [col], 28, 1e-300, 5)
        lo, hi = a.csc_ptr[col], a.csc_ptr[col + 1]
        for p in range(lo, hi):
            pcol[p] = contrib.get(int(a.csc_rows[p]), 0.0)
    return pcol


def _worker(rank, world, port_no, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = golden_io.load(name)
        a = c.sa
        t = port.transition_tables(a)
        ni = port.allocate(t, 20 * c.n)
        pre = np.concatenate([[0], np.cumsum(ni)])
        z = port.zeta_prefix("exponential", 30)
        r = a.scipy_csr() @ np.ones(c.n)
        # action: q over my (walk-balanced) column shard, all-gathered by range
        shards = parallel.column_shards(pre, world)
        cb, ce = shards[rank]
        cols = [j for j in range(cb, ce) if ni[j] > 0]
        qd, _ = port.action_columns(t, r, z, ni, cols, 28, 1e-300, 5)
        q = torch.zeros(c.n, dtype=torch.float64)
        for j, val in qd.items():
            q[j] = val
        parallel.gather_ranges(q, [shards[0][0]] + [b for _, b in shards])
        # diag: per-entry partials of my (cost-balanced) column shard = one
        # contiguous CSC range, all-gathered; then d by row shard
        cost = column_costs_np(a.csc_ptr, a.csc_rows, a.row_ptr, ni, 28)
        dsh = parallel.column_shards(pre, world, cost)
        dcols = [j for j in range(*dsh[rank]) if ni[j] > 0]
        pcol = torch.from_numpy(_per_entry_partials(c, t, z, ni, dcols))
        cuts = a.csc_ptr[[dsh[0][0]] + [b for _, b in dsh]]
        parallel.gather_ranges(pcol, cuts)
        if rank == 0:
            out.put((q.numpy().copy(), pcol.numpy().copy(), shards, dsh))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["er300", "kron8"])
def test_sharded_assembly_matches_single_process(name):
    ctx = tmp.get_context("spawn")
    out = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, name, out)) for r in range(2)]
    for p in procs:
        p.start()
    q, pcol, shards, dsh = out.get(timeout=400)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = golden_io.load(name)
    t = port.transition_tables(c.sa)
    ni = port.allocate(t, 20 * c.n)
    z = port.zeta_prefix("exponential", 30)
    r = c.sa.scipy_csr() @ np.ones(c.n)
    cols = np.flatnonzero(ni)
    qd, _ = port.action_columns(t, r, z, ni, cols, 28, 1e-300, 5)
    q1 = np.zeros(c.n)
    for j, val in qd.items():
        q1[j] = val
    assert np.array_equal(q, q1)
    p1 = _per_entry_partials(c, t, z, ni, cols)
    assert np.array_equal(pcol, p1)
    # shards: contiguous, cover all columns; walk shards balanced by walks
    for sh in (shards, dsh):
        assert sh[0][0] == 0 and sh[0][1] == sh[1][0] and sh[1][1] == c.n
    pre = np.concatenate([[0], np.cumsum(ni)])
    w0 = pre[shards[0][1]] - pre[shards[0][0]]
    assert abs(w0 - pre[-1] / 2) <= ni.max()


def _rmat_csr(scale, ef, seed=0, pa=0.57, pb=0.19, pc=0.19):
    """Small symmetrised R-MAT (graphgen.py:138-143 quadrant rule), numpy."""
    rng = np.random.default_rng(seed)
    m = ef << scale
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for _ in range(scale):
        x = rng.random(m)
        rb = x >= pa + pb
        cb = ((x >= pa) & ~rb) | (x >= pa + pb + pc)
        u = (u << 1) | rb
        v = (v << 1) | cb
    keep = u != v
    u, v = u[keep], v[keep]
    n = 1 << scale
    key = np.unique(np.concatenate([(u << scale) | v, (v << scale) | u]))
    rows, cols = key >> scale, key & (n - 1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return n, row_ptr, cols


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_cost_balanced_shards_hub_heavy(parts):
    """On a hub-heavy R-MAT the diag cost of contiguous shards is within 10%
    of the mean, while equal-walk shards put most of it on the hub ranks."""
    n, row_ptr, cols = _rmat_csr(14, 16)
    deg = np.diff(row_ptr)
    p = np.sqrt(deg) / np.sqrt(deg).sum()  # ||C_j||_2 of a 0/1 matrix
    ni = port.largest_remainder(p, 200 * n)
    pre = np.concatenate([[0], np.cumsum(ni)])
    cost = column_costs_np(row_ptr, cols, row_ptr, ni, 23)
    cp = np.concatenate([[0], np.cumsum(cost)])
    sh = parallel.column_shards(pre, parts, cost)
    per = np.array([cp[b] - cp[a] for a, b in sh], dtype=np.float64)
    assert np.max(np.abs(per / per.mean() - 1)) < 0.10, per / per.mean()
    naive = parallel.column_shards(pre, parts)
    pn = np.array([cp[b] - cp[a] for a, b in naive], dtype=np.float64)
    assert pn.max() / pn.mean() > per.max() / per.mean()
    # the torch (device-style) search gives the same cuts
    assert parallel.column_shards(torch.tensor(pre), parts, torch.tensor(cost)) == sh


def test_column_shards_device_free_cases():
    pre = np.array([0, 0, 5, 5, 5, 9, 20, 20])
    for parts in (1, 2, 3, 4, 8):
        sh = parallel.column_shards(pre, parts)
        assert sh[0][0] == 0 and sh[-1][1] == 7
        assert all(a[1] == b[0] for a, b in zip(sh[:-1], sh[1:]))
        assert all(a <= b for a, b in sh)
        assert sum(parallel.shard_walks(pre, sh)) == 20
    assert parallel.row_shards(10, 3) == [(0, 3), (3, 6), (6, 10)]
    sh_t = parallel.column_shards(torch.tensor(pre), 3)
    assert sh_t == parallel.column_shards(pre, 3)
