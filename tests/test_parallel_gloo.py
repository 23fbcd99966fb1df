"""Multi-process host logic of the column-sharded path (parallel.py), world
size 2 over gloo on CPU.  The per-column compute is the oracle (test-only
stand-in for the device); what is under test is the sharding and the exact
assembly: sharded results must equal the single-process result bit for bit."""
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


def _worker(rank, world, port_no, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = golden_io.load(name)
        t = port.transition_tables(c.sa)
        ni = port.allocate(t, 20 * c.n)
        pre = np.concatenate([[0], np.cumsum(ni)])
        z = port.zeta_prefix("exponential", 30)
        r = c.sa.scipy_csr() @ np.ones(c.n)
        # action: q over my column shard, zeros elsewhere, assembled exactly
        cb, ce = parallel.column_shards(pre, world)[rank]
        cols = [j for j in range(cb, ce) if ni[j] > 0]
        qd, _ = port.action_columns(t, r, z, ni, cols, 28, 1e-300, 5)
        q = torch.zeros(c.n, dtype=torch.float64)
        for j, val in qd.items():
            q[j] = val
        parallel.assemble(q)
        # diag: Eq. 20 contributions of my columns, assembled exactly
        dd, _ = port.diag_columns(c.sa, t, z, ni, cols, 28, 1e-300, 5)
        d = torch.zeros(c.n, dtype=torch.float64)
        for i, val in dd.items():
            d[i] = val
        parallel.assemble(d)
        if rank == 0:
            out.put((q.numpy().copy(), d.numpy().copy(), parallel.column_shards(pre, world)))
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
    q, d, shards = out.get(timeout=240)
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
    dd, _ = port.diag_columns(c.sa, t, z, ni, cols, 28, 1e-300, 5)
    assert np.array_equal(q, q1)
    # diag contributions of two shards are summed per row: rows touched by both
    # shards differ only by summation order
    d1 = np.zeros(c.n)
    for i, val in dd.items():
        d1[i] = val
    np.testing.assert_allclose(d, d1, rtol=1e-13, atol=1e-300)
    # shards: contiguous, cover all columns, balanced by walks
    assert shards[0][0] == 0 and shards[0][1] == shards[1][0] and shards[1][1] == c.n
    pre = np.concatenate([[0], np.cumsum(ni)])
    w0 = pre[shards[0][1]] - pre[shards[0][0]]
    assert abs(w0 - pre[-1] / 2) <= ni.max()


def test_column_shards_device_free_cases():
    pre = np.array([0, 0, 5, 5, 5, 9, 20, 20])
    for parts in (1, 2, 3, 4, 8):
        sh = parallel.column_shards(pre, parts)
        assert sh[0][0] == 0 and sh[-1][1] == 7
        assert all(a[1] == b[0] for a, b in zip(sh[:-1], sh[1:]))
        assert all(a <= b for a, b in sh)
    assert parallel.row_shards(10, 3) == [(0, 3), (3, 6), (6, 10)]
    sh_t = parallel.column_shards(torch.tensor(pre), 3)
    assert sh_t == parallel.column_shards(pre, 3)
