"""The peer-memory exchanges (parallel.sharded_action_peer / mcf_spmv_peer,
parallel.sharded_diag_peer / mcf_diag_combine_peer) with world size 2.  Two processes share ONE GPU here (the
sandbox has one): CUDA IPC between processes on a device is the same mapping
path as between GPUs of a node, the kernels never wait on each other (host
barriers only), and this checks results, not speed.  y and d must equal the
single-process estimates bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as tmp

from tests import golden_io

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _as_matrix(a, symmetric):
    from scipy import sparse

    class M:
        pass
    m = M()
    m.csr = sparse.csr_array((a.vals, a.col_ids.astype(np.int32), a.row_ptr), shape=(a.n, a.n))
    m.csc = sparse.csc_array((a.csc_vals, a.csc_rows.astype(np.int32), a.csc_ptr), shape=(a.n, a.n))
    m.symmetric_hint = symmetric
    return m


def _worker(rank, world, port_no, name, n_walks, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_01037_b200 as mc
        from paper_2308_01037_b200 import parallel
        c = golden_io.load(name)
        g = mc.DeviceGraph(_as_matrix(c.sa, c.symmetric), gamma=0.05)
        y, st = parallel.sharded_action_peer(g, mc.EXPONENTIAL, None, mc.WalkConfig(n_walks, 1e-6, 28, 11))
        d, sd = parallel.sharded_diag_peer(g, mc.EXPONENTIAL, mc.WalkConfig(n_walks, 1e-6, 28, 12))
        emitted = torch.tensor([int(st[1]), int(sd[1])])
        dist.all_reduce(emitted)
        if rank == 0:
            out.put((y.cpu().numpy(), d.cpu().numpy(), emitted.tolist()))
        g.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("units", [None, "split"])
@pytest.mark.parametrize("name", ["ba400", "kron8"])
def test_peer_exchange_matches_single_process(name, units, monkeypatch):
    """units="split": the diag combine by key-group units (forced on these
    small graphs, every column split, narrow-column tiers) on each rank's
    column shard; the spawned ranks inherit the environment."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if units:
        monkeypatch.setenv("MCF_DIAG_UNITS", "1")
        monkeypatch.setenv("MCF_UNIT_SMALL_NEED", "64")
        monkeypatch.setenv("MCF_UNIT_SMALL_CUT", "32")
    import paper_2308_01037_b200 as mc
    c = golden_io.load(name)
    n_walks = 50 * c.n
    ctx = tmp.get_context("spawn")
    out = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, name, n_walks, out)) for r in range(2)]
    for p in procs:
        p.start()
    y2, d2, em2 = out.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = mc.DeviceGraph(_as_matrix(c.sa, c.symmetric), gamma=0.05)
    ref = mc.rand_funm_action(g, mc.EXPONENTIAL, None, mc.WalkConfig(n_walks, 1e-6, 28, 11))  # v = 1 as the shards
    refd = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(n_walks, 1e-6, 28, 12))
    assert em2 == [ref.emissions, refd.emissions]
    assert np.array_equal(y2, np.asarray(ref.values))
    assert np.array_equal(d2, np.asarray(refd.values))


def _worker_big(rank, world, port_no, name, n_walks, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2308_01037_b200 as mc
        from paper_2308_01037_b200 import parallel
        c = golden_io.load(name)
        g = mc.DeviceGraph(_as_matrix(c.sa, c.symmetric), gamma=0.05)
        cfg = mc.WalkConfig(n_walks, 1e-6, 28, 21)
        y, st = parallel.sharded_action(g, mc.EXPONENTIAL, None, cfg)        # NCCL-style all-gather path (gloo here)
        d, sd = parallel.sharded_diag(g, mc.EXPONENTIAL, mc.WalkConfig(50 * c.n, 1e-6, 28, 22))
        emitted = torch.tensor([int(st[1]), int(sd[1])])
        dist.all_reduce(emitted)
        if rank == 0:
            out.put((y.cpu().numpy(), d.cpu().numpy(), emitted.tolist()))
        g.close()
    finally:
        dist.destroy_process_group()


def test_action_beyond_2_31_walks_single_and_two_ranks():
    """N_s > 2^31 walks (the reference has no cap, walker.py:55, :263): one
    process runs them in column batches inside mcf_funm_action; two ranks
    each get a cost-balanced shard with its own walk capacity.  q / y equal
    the explicit per-half launches, and 1 vs 2 ranks, bit for bit; the diag
    all-gather path (per-entry partials of each rank's CSC range) as well."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2308_01037_b200 as mc
    from paper_2308_01037_b200.device import WalkParams
    name = "ba400"
    c = golden_io.load(name)
    n_walks = (1 << 31) + 12_345_678
    g = mc.DeviceGraph(_as_matrix(c.sa, c.symmetric), gamma=0.05)
    cfg = mc.WalkConfig(n_walks, 1e-6, 28, 21)
    ref = mc.rand_funm_action(g, mc.EXPONENTIAL, None, cfg)   # one call: batched inside the library
    assert ref.walks == n_walks
    # the same walks as two explicit column halves (each < 2^31 walks)
    z = mc.EXPONENTIAL.prefix(30)
    ni, pre = g.allocate(n_walks)
    half = int(torch.searchsorted(pre, pre[-1] // 2).item())
    q = torch.zeros(g.n, dtype=torch.float64, device="cuda")
    r = ref.aux["r"]  # the row sums the one-call path used (mcf_spmv's long rows sum in another order)
    st = g.new_stats()
    params = WalkParams(cfg, z)
    for cols in ((0, half), (half, g.n)):
        cap = int(pre[cols[1]] - pre[cols[0]])
        assert cap < (1 << 31)
        g.walk_action(params.derive(capacity=cap), pre, r, q, cols=cols, stats=st)
    assert np.array_equal(q.cpu().numpy(), ref.aux["q"].cpu().numpy())
    refd = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(50 * c.n, 1e-6, 28, 22))
    ctx = tmp.get_context("spawn")
    out = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker_big, args=(k, 2, port_no, name, n_walks, out)) for k in range(2)]
    for p in procs:
        p.start()
    y2, d2, em2 = out.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert em2 == [ref.emissions, refd.emissions]
    assert np.array_equal(y2, np.asarray(ref.values))
    assert np.array_equal(d2, np.asarray(refd.values))
