"""Device parity against the reference (golden fixtures) and the CPU oracle.

Bar (BASELINE.json north_star): replaying the reference's own sampled entry
stream reproduces its estimates to 1e-10 relative (fp64); integer work (walk
budgets, emission / truncation counts) is bit-exact; the device transition
tables equal the reference's bit for bit."""
import numpy as np
import pytest
from scipy import sparse

from oracle import port
from tests import golden_io

pytestmark = pytest.mark.gpu

REL = 1e-10  # replay tolerance stated by the north star


@pytest.fixture(scope="module", params=["compact", "fat"])
def layout(request):
    """Both walk layouts (MCF_WALK_LAYOUT is read when a graph is built)."""
    import os
    old = os.environ.get("MCF_WALK_LAYOUT")
    os.environ["MCF_WALK_LAYOUT"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("MCF_WALK_LAYOUT", None)
    else:
        os.environ["MCF_WALK_LAYOUT"] = old


@pytest.fixture(scope="module")
def mc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2308_01037_b200 as m
    return m


def as_matrix(a: port.Csr, symmetric=False):
    class M:
        pass
    m = M()
    m.csr = sparse.csr_array((a.vals, a.col_ids.astype(np.int32), a.row_ptr), shape=(a.n, a.n))
    m.csc = sparse.csc_array((a.csc_vals, a.csc_rows.astype(np.int32), a.csc_ptr), shape=(a.n, a.n))
    m.symmetric_hint = symmetric
    return m


def rel_err(x, ref):
    x, ref = np.asarray(x), np.asarray(ref)
    scale = np.maximum(np.abs(ref), 1e-300)
    return float(np.max(np.abs(x - ref) / scale))


@pytest.mark.parametrize("name", golden_io.CASES)
def test_device_tables_bitwise(mc, name):
    c = golden_io.load(name)
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric))
    t = {k: v.cpu().numpy() for k, v in g.tables().items()}
    assert np.array_equal(t["row_abs_sum"], c["m_row_abs_sum"])
    assert np.array_equal(t["col_norms"], c["m_col_norms"])
    assert np.array_equal(t["init_prob"], c["m_init_prob"])
    assert g.info["max_row_abs_sum"] ** 2 == float(c["alpha"])


@pytest.fixture(params=["fused", "passes"])
def alloc_path(request):
    """Both budget implementations: the persistent one-kernel path (n up to
    sm_count * 8192) and the multi-pass path used beyond that."""
    import os
    old = os.environ.get("MCF_ALLOC_PATH")
    os.environ["MCF_ALLOC_PATH"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("MCF_ALLOC_PATH", None)
    else:
        os.environ["MCF_ALLOC_PATH"] = old


@pytest.mark.parametrize("name", golden_io.CASES)
def test_device_allocation_bitwise(mc, alloc_path, name):
    c = golden_io.load(name)
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric))
    for ns in (1, 7, 1000, 12345, 10 * c.n + 3):
        ni, pre = g.allocate(ns)
        assert np.array_equal(ni.cpu().numpy(), c[f"ni_{ns}"]), ns
        assert int(pre[-1]) == ns
        assert np.array_equal(pre.cpu().numpy(), np.concatenate([[0], np.cumsum(c[f"ni_{ns}"])]))


def test_allocation_large_both_paths(mc, alloc_path):
    """BA n = 1e6 (config 2): budgets equal the reference rule on the device
    p for tie-heavy and tie-free budgets, and walk_pre is their prefix sum."""
    from paper_2308_01037_b200 import graphs
    g = mc.DeviceGraph(graphs.barabasi_albert(1_000_000, 4, seed=0))
    p = g.tables()["init_prob"].cpu().numpy()
    for ns in (640_000, 1, 999_999, 1_000_003, 12_345_679, 3 * 10**7 + 11):
        ni, pre = g.allocate(ns)
        ref = port.largest_remainder(p, ns)
        assert np.array_equal(ni.cpu().numpy(), ref), ns
        assert np.array_equal(pre.cpu().numpy(), np.concatenate([[0], np.cumsum(ref)])), ns


@pytest.mark.parametrize("name", golden_io.CASES)
def test_replay_matches_reference(mc, layout, name):
    c = golden_io.load(name)
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric))
    assert g.info["walk_layout"] == (1 if layout == "fat" else 0)
    for j, r in enumerate(c.runs):
        p = f"r{j}_"
        cfg = mc.WalkConfig(r["n_walks"], r["cutoff"], r["max_steps"], r["seed"])
        if r["mode"] == "action":
            out = mc.rand_funm_action(g, r["tag"], c[p + "v"], cfg, replay=c.record(j))
            assert rel_err(out.values, c[p + "y"]) < REL
            assert rel_err(out.aux["q"].cpu().numpy(), c[p + "q"]) < REL or np.allclose(
                out.aux["q"].cpu().numpy(), c[p + "q"], rtol=REL, atol=1e-300)
        else:
            out = mc.rand_funm_diag(g, r["tag"], cfg, replay=c.record(j))
            assert rel_err(out.values, c[p + "d"]) < REL
        assert out.emissions == int(c[p + "emissions"])
        assert out.truncated == int(c[p + "truncated"])
        assert out.walks == r["n_walks"]


@pytest.mark.parametrize("name", golden_io.CASES)
def test_unit_combine_replay_golden(mc, name, monkeypatch):
    """The unit combine (the default above the dense-Q size) forced onto the
    golden graphs: dense one-unit tables, hashed one-unit tables and columns
    split into up to 128 key-group units all replay the reference's streams to
    1e-10, bit-identical to the single-table combine."""
    c = golden_io.load(name)
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric))
    for j, r in enumerate(c.runs):
        if r["mode"] != "diag":
            continue
        p = f"r{j}_"
        cfg = mc.WalkConfig(r["n_walks"], r["cutoff"], r["max_steps"], r["seed"])
        monkeypatch.setenv("MCF_DIAG_UNITS", "0")
        ref = mc.rand_funm_diag(g, r["tag"], cfg, replay=c.record(j)).values
        for env in ({"MCF_DIAG_UNITS": "1"}, {"MCF_DIAG_UNITS": "1", "MCF_UNIT_SMALL_NEED": "64"},
                    {"MCF_DIAG_UNITS": "1", "MCF_UNIT_SMALL_NEED": "8", "MCF_UNIT_CHUNK": "32"},
                    {"MCF_DIAG_UNITS": "1", "MCF_UNIT_SMALL_NEED": "64", "MCF_UNIT_PARTITION": "0"}):
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            out = mc.rand_funm_diag(g, r["tag"], cfg, replay=c.record(j))
            for k in env:
                monkeypatch.delenv(k)
            assert rel_err(out.values, c[p + "d"]) < REL, env
            assert np.array_equal(out.values, ref), env  # (weighted graphs: the single-table path both times)


def test_replay_rejects_corrupt_stream(mc):
    c = golden_io.load("signed6")
    g = mc.DeviceGraph(as_matrix(c.sa))
    r = c.runs[0]
    rec = c.record(0)
    bad = port.Record(rec.walk_pre, rec.walk_off.copy(), rec.entries.copy())
    bad.walk_off[1:] += 1  # walk 0 claims an extra entry it never consumes
    bad.entries = np.concatenate([bad.entries[:1], bad.entries])
    cfg = mc.WalkConfig(r["n_walks"], r["cutoff"], r["max_steps"], r["seed"])
    with pytest.raises(mc.ArgumentError):
        mc.rand_funm_action(g, r["tag"], c["r0_v"], cfg, replay=bad)


def test_replay_oracle_stream_er2000(mc):
    """Larger case recorded at test time by the oracle (config-1 shape, ER LCC)."""
    rng = np.random.default_rng(4)
    n = 2000
    u, v = rng.integers(0, n, 8000), rng.integers(0, n, 8000)
    keep = u != v
    m = sparse.coo_array((np.ones(keep.sum() * 2), (np.r_[u[keep], v[keep]], np.r_[v[keep], u[keep]])), shape=(n, n))
    m = sparse.csr_array(m)
    m.data[:] = 1.0
    m.sum_duplicates()
    m.data[:] = 1.0
    a = port.Csr.from_any(m)
    lam = float(np.max(np.linalg.eigvalsh(m.toarray())))
    a = a.scaled(1.0 / lam)
    g = mc.DeviceGraph(as_matrix(a, True))
    for mode in ("action", "diag"):
        if mode == "action":
            run = port.funm_action(a, "exponential", np.ones(n), 20 * n, 1e-300, 28, 0, record=True)
            out = mc.rand_funm_action(g, "exponential", np.ones(n), mc.WalkConfig(20 * n, 1e-300, 28, 0),
                                      replay=run.record)
        else:
            run = port.funm_diag(a, "exponential", 20 * n, 1e-300, 28, 0, record=True)
            out = mc.rand_funm_diag(g, "exponential", mc.WalkConfig(20 * n, 1e-300, 28, 0), replay=run.record)
        assert rel_err(out.values, run.payload) < REL
        assert out.emissions == run.emissions


@pytest.mark.parametrize("m_steps", [1, 5, 28])
def test_truncation_mapping_kat_device(mc, m_steps):
    """gamma*[[0,1],[1,0]]: deterministic walks -> exactly dense_funm(terms=M+1)."""
    for gam in (0.5, 0.9):
        a = mc.SparseMatrix.from_dense([[0, gam], [gam, 0]], True)
        ref = port.dense_funm(port.Csr.from_dense([[0, gam], [gam, 0]]), "exponential", m_steps + 1)
        cfg = mc.WalkConfig(64, 1e-300, m_steps, 3)
        d = mc.rand_funm_diag(a, mc.EXPONENTIAL, cfg)
        y = mc.rand_funm_action(a, mc.EXPONENTIAL, np.ones(2), cfg)
        np.testing.assert_allclose(d.values, np.diag(ref), rtol=4e-15)
        np.testing.assert_allclose(y.values, ref.sum(1), rtol=4e-15)
        assert d.truncated == 64 and y.emissions == 64 * m_steps


def test_spec_closed_forms_device(mc):
    """zero-variance involutory graph."""
    a = mc.SparseMatrix.from_dense([[0, 1], [1, 0]], True)
    cfg = mc.WalkConfig(10**6, 1e-10, 10_000, 0)
    rep = mc.total_communicability(a, 0.1, cfg)
    np.testing.assert_allclose(rep.scores, np.exp(0.1), rtol=5e-3)
    rep = mc.subgraph_centrality(a, 0.1, cfg)
    np.testing.assert_allclose(rep.scores, np.cosh(0.1), rtol=5e-3)
    k = mc.katz_centrality(a, 0.5, mc.WalkConfig(10**5, 1e-10, 10_000, 0), gamma=0.5)
    np.testing.assert_allclose(k.scores, [2.0, 2.0], rtol=5e-3)
    kc = mc.katz_centrality(a, 0.5, None, method="cg", gamma=0.5)
    np.testing.assert_allclose(kc.scores, [2.0, 2.0], rtol=1e-9)


def test_self_loop_and_absorbing_kats(mc):
    # self loop 0.5, W_c = 0.1 -> 4 emissions
    a = mc.SparseMatrix.from_dense([[0.5]])
    y = mc.rand_funm_action(a, mc.EXPONENTIAL, np.ones(1), mc.WalkConfig(1, 0.1, 100, 0))
    assert y.emissions == 4 and y.truncated == 0
    # absorbing start column: single emission then terminal
    b = mc.SparseMatrix.from_dense([[0, 0], [1, 0]])
    y = mc.rand_funm_action(b, mc.EXPONENTIAL, np.ones(2), mc.WalkConfig(5, 1e-6, 100, 0))
    assert y.emissions == 5 and y.absorbed == 5


def test_degenerate_and_argument_errors(mc):
    with pytest.raises(mc.DegenerateInputError):
        mc.DeviceGraph(mc.SparseMatrix(sparse.csr_array((3, 3)), sparse.csc_array((3, 3))))
    a = mc.SparseMatrix.from_dense([[0, 1], [1, 0]], True)
    with pytest.raises(mc.ArgumentError):
        mc.rand_funm_action(a, mc.EXPONENTIAL, np.ones(3), mc.WalkConfig(10))
    with pytest.raises(mc.ArgumentError):
        mc.subgraph_centrality(mc.SparseMatrix.from_dense([[0, 1], [0, 0]]), 0.1, mc.WalkConfig(10))


def test_fat_and_compact_layouts_agree_bitwise(mc):
    """The layout changes which memory a step reads, never the walk."""
    import os
    c = golden_io.load("ba400")
    out = {}
    for lay in ("compact", "fat"):
        os.environ["MCF_WALK_LAYOUT"] = lay
        g = mc.DeviceGraph(as_matrix(c.sa, True))
        cfg = mc.WalkConfig(50_000, 1e-6, 28, 3)
        out[lay] = (mc.rand_funm_action(g, mc.EXPONENTIAL, np.linspace(0, 1, c.n), cfg).values,
                    mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values)
    os.environ.pop("MCF_WALK_LAYOUT", None)
    assert np.array_equal(out["compact"][0], out["fat"][0])
    assert np.array_equal(out["compact"][1], out["fat"][1])


def test_determinism_and_partition_invariance(mc):
    import torch
    c = golden_io.load("kron8")
    g = mc.DeviceGraph(as_matrix(c.sa, True))
    cfg = mc.WalkConfig(50_000, 1e-300, 23, 9)
    from paper_2308_01037_b200.device import WalkParams
    z = mc.EXPONENTIAL.prefix(cfg.max_steps + 2)
    p = WalkParams(cfg, z, g.device)
    ni, pre = g.allocate(cfg.n_walks)
    r = g.spmv(torch.ones(g.n, dtype=torch.float64, device=g.device))
    outs = []
    for cuts in ([0, g.n], [0, 57, g.n], [0, 3, 100, 101, g.n]):
        q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
        pc = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            g.walk_action(p, pre, r, q, cols=(lo, hi), stats=g.new_stats())
            g.walk_diag(p, pre, pc, cols=(lo, hi), stats=g.new_stats())
        outs.append((q.cpu().numpy(), g.diag_combine(z[0], z[1], pc).cpu().numpy()))
    for q, d in outs[1:]:
        assert np.array_equal(q, outs[0][0])
        assert np.array_equal(d, outs[0][1])


def _z_check(z, n):
    from scipy.stats import norm
    bound = norm.isf(0.01 / (2 * n))  # Bonferroni
    assert np.mean(np.abs(z) <= 3) >= 0.99, np.sort(np.abs(z))[-10:]
    assert np.max(np.abs(z)) <= bound + 0.5, (np.max(np.abs(z)), bound)
    assert abs(np.mean(z)) < 0.15 and 0.8 < np.std(z) < 1.2, (np.mean(z), np.std(z))


def test_device_rng_action_statistics(mc, layout):
    """Device RNG vs exact 30-term Taylor action (SURVEY.md §4 z-test recipe)."""
    c = golden_io.load("ba400")
    g = mc.DeviceGraph(as_matrix(c.sa, True))
    cfg = mc.WalkConfig(400 * 5000, 1e-300, 28, 123)
    y = mc.rand_funm_action(g, mc.EXPONENTIAL, np.ones(c.n), cfg, stderr=True)
    exact = port.taylor_action(c.sa, "exponential", np.ones(c.n), 29)
    _z_check((y.values - exact) / y.stderr, c.n)


def test_device_rng_diag_statistics(mc):
    """Device RNG diag vs exact truncated series, SE from independent replicas."""
    c = golden_io.load("er300")
    g = mc.DeviceGraph(as_matrix(c.sa, True))
    exact = np.diag(port.dense_funm(c.sa, "exponential", 29))
    reps = np.array([mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(300 * 400, 1e-300, 28, s)).values
                     for s in range(32)])
    z = (reps.mean(0) - exact) / (reps.std(0, ddof=1) / np.sqrt(reps.shape[0]))
    assert np.mean(np.abs(z) <= 3.5) >= 0.98
    assert abs(np.mean(z)) < 0.3


def test_device_rng_weighted_signed_rows(mc, layout):
    """Non-uniform rows (inverse-CDF path) and negative values (packed signs)."""
    c = golden_io.load("signed6")
    g = mc.DeviceGraph(as_matrix(c.sa))
    exact = port.taylor_action(c.sa, "exponential", np.ones(c.n), 41)
    reps = np.array([mc.rand_funm_action(g, mc.EXPONENTIAL, np.ones(c.n), mc.WalkConfig(200_000, 1e-300, 40, s))
                     .values for s in range(16)])
    sd = reps.std(0, ddof=1)
    fixed = sd == 0  # absorbing row 4: y_4 = v_4 with no walk contribution
    assert fixed.sum() == 1 and np.allclose(reps.mean(0)[fixed], exact[fixed], rtol=1e-14)
    z = (reps.mean(0)[~fixed] - exact[~fixed]) / (sd[~fixed] / 4.0)
    assert np.all(np.abs(z) < 5), z


def test_katz_resolvent_statistics(mc):
    c = golden_io.load("sw64_katz")
    a = as_matrix(c.a, True)
    gam = c.gamma
    exact = port.cg_solve(c.a, gam, np.ones(c.n), tol=1e-13)
    rep = mc.katz_centrality(a, 0.85, mc.WalkConfig(10**6, 1e-8, 10_000, 1), stderr=True)
    assert rep.gamma == pytest.approx(gam, rel=1e-15)
    z = (rep.scores - exact) / rep.result.stderr
    assert np.max(np.abs(z)) < 5


@pytest.mark.parametrize("seed", [0, 1])
def test_device_tables_bitwise_hub_rows(mc, seed):
    """Rows/columns far longer than the warp-per-row thresholds (64 / 256),
    random signed weights, non-symmetric: tables still equal the oracle's
    (which is pinned to the reference) bit for bit, and so do the budgets."""
    import torch
    rng = np.random.default_rng(seed)
    n = 3001
    rows, cols = [], []
    for hub, deg in ((0, 3000), (7, 1500), (100, 300), (2999, 70), (50, 129), (60, 140), (70, 200), (80, 250),
                     (90, 256), (95, 257), (97, 1030)):
        nb = rng.choice(n, deg, replace=False)
        rows += [hub] * deg
        cols += list(nb)
        rows += list(nb)
        cols += [hub] * deg
    r = rng.integers(0, n, 20000)
    c = rng.integers(0, n, 20000)
    m = sparse.coo_array((rng.normal(size=len(rows) + r.size), (np.r_[rows, r], np.r_[cols, c])), shape=(n, n)).tocsr()
    m.sum_duplicates()
    m.data[m.data == 0] = 0.5
    m.sort_indices()
    a = port.Csr.from_any(m)
    t = port.transition_tables(a)
    g = mc.DeviceGraph(as_matrix(a))
    d = {k: v.cpu().numpy() for k, v in g.tables().items()}
    assert np.array_equal(d["row_abs_sum"], t.rsum)
    assert np.array_equal(d["col_norms"], t.col_norms)
    assert np.array_equal(d["init_prob"], t.init_prob)
    for ns in (1000, 77777):
        assert np.array_equal(g.allocate(ns)[0].cpu().numpy(), port.allocate(t, ns))
    x = rng.normal(size=n)
    y = g.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_allclose(y, m @ x, rtol=1e-12, atol=1e-12)


def test_entry_and_mc_replay_parity(mc):
    """rand_funm_entry and mc_baseline replaying oracle-recorded streams."""
    c = golden_io.load("ba400")
    g = mc.DeviceGraph(as_matrix(c.sa, True))
    hub = int(np.argmax(np.diff(c.sa.row_ptr)))
    v = np.linspace(0.5, 1.5, c.n)
    run = port.funm_entry(c.sa, "exponential", v, hub, 20_000, 1e-6, 28, 4, record=True)
    out = mc.rand_funm_entry(g, mc.EXPONENTIAL, v, hub, mc.WalkConfig(20_000, 1e-6, 28, 4), replay=run.record)
    assert rel_err(out.values, run.payload) < REL and out.emissions == run.emissions
    for mode in ("diag", "action"):
        run = port.mc_baseline(c.sa, "exponential", 20, 1e-6, 28, 5, mode, v=v, record=True)
        out = mc.mc_baseline(g, mc.EXPONENTIAL, mc.WalkConfig(20, 1e-6, 28, 5), mode, v=v, replay=run.record)
        assert rel_err(out.values, run.payload) < REL
        assert out.emissions == run.emissions


def test_entry_device_rng_matches_exact(mc):
    c = golden_io.load("er300")
    g = mc.DeviceGraph(as_matrix(c.sa, True))
    exact = port.taylor_action(c.sa, "exponential", np.ones(c.n), 29)
    for i in (0, 17, 123):
        ys = [mc.rand_funm_entry(g, mc.EXPONENTIAL, np.ones(c.n), i, mc.WalkConfig(200_000, 1e-300, 28, s)).values[0]
              for s in range(8)]
        z = (np.mean(ys) - exact[i]) / (np.std(ys, ddof=1) / np.sqrt(8))
        assert abs(z) < 5, (i, z)
    e = mc.rand_funm_entry(g, mc.EXPONENTIAL, np.ones(c.n), 5, mc.WalkConfig(1000))
    assert e.walks == 1000


def test_mc_baseline_dominated_by_rand_funm_diag(mc):
    """SPEC acceptance 6 (§4.2 claim): at equal global walk budget on a 64-node
    small world, rand_funm_diag beats mc_baseline(diag) in l_inf error in >= 8/10 seeds."""
    c = golden_io.load("sw64_katz")
    a = c.a.scaled(1e-1)
    g = mc.DeviceGraph(as_matrix(a, True))
    exact = np.diag(port.dense_funm(a, "exponential", 40))
    wins = 0
    for s in range(10):
        d1 = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(64 * 1000, 1e-10, 100, s)).values
        d0 = mc.mc_baseline(g, mc.EXPONENTIAL, mc.WalkConfig(1000, 1e-10, 100, s), "diag").values
        wins += np.max(np.abs(d1 - exact)) < np.max(np.abs(d0 - exact))
    assert wins >= 8


def _hub_graph(seed=0, n=5000, hub_deg=4000):
    rng = np.random.default_rng(seed)
    nb = rng.choice(np.arange(1, n), hub_deg, replace=False)
    u = np.r_[np.zeros(hub_deg, dtype=np.int64), rng.integers(0, n, 6 * n)]
    v = np.r_[nb, rng.integers(0, n, 6 * n)]
    keep = u != v
    m = sparse.coo_array((np.ones(2 * keep.sum()), (np.r_[u[keep], v[keep]], np.r_[v[keep], u[keep]])), shape=(n, n))
    m = sparse.csr_array(m)
    m.sum_duplicates()
    m.data[:] = 1.0
    a = port.Csr.from_any(m)
    lam = float(np.max(np.linalg.eigvalsh(m.toarray()))) if n <= 3000 else float(
        __import__("scipy.sparse.linalg", fromlist=["eigsh"]).eigsh(m.astype(float), k=1, which="LA",
                                                                      v0=np.ones(n))[0][0])
    return a.scaled(1.0 / lam)


def test_diag_hub_push_path_bitwise_and_replay(mc):
    """Hub rows (degree >= 2048) take the bitmap push path on uniform-value
    graphs; fixed-point sums make it bitwise equal to the pull path, and replay
    still matches the oracle to 1e-10."""
    import os
    a = _hub_graph()
    cfg = mc.WalkConfig(5000 * 30, 1e-300, 20, 2)
    outs = []
    for mb in (None, "0"):
        if mb is None:
            os.environ.pop("MCF_HUB_BITMAP_MB", None)
        else:
            os.environ["MCF_HUB_BITMAP_MB"] = mb
        g = mc.DeviceGraph(as_matrix(a, True))
        outs.append(mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values)
    os.environ.pop("MCF_HUB_BITMAP_MB", None)
    assert np.array_equal(outs[0], outs[1])
    run = port.funm_diag(a, "exponential", 5000 * 4, 1e-300, 20, 3, record=True)
    g = mc.DeviceGraph(as_matrix(a, True))
    out = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(5000 * 4, 1e-300, 20, 3), replay=run.record)
    assert rel_err(out.values, run.payload) < REL


def _multi_hub_graph(seed=0, n=40000, hub_degs=(1500, 3000, 6000, 12000, 24000)):
    """Uniform-value graph above the dense-Q size with hubs of several degrees,
    so the hub columns' Q_c need clusters of 2, 4 and 8 CTAs (and one a global
    table)."""
    rng = np.random.default_rng(seed)
    us, vs = [rng.integers(0, n, 6 * n)], [rng.integers(0, n, 6 * n)]
    for h, d in enumerate(hub_degs):
        us.append(np.full(d, h, dtype=np.int64))
        vs.append(rng.choice(np.arange(len(hub_degs), n), d, replace=False))
    u, v = np.concatenate(us), np.concatenate(vs)
    keep = u != v
    m = sparse.coo_array((np.ones(2 * keep.sum()), (np.r_[u[keep], v[keep]], np.r_[v[keep], u[keep]])), shape=(n, n))
    m = sparse.csr_array(m)
    m.sum_duplicates()
    m.data[:] = 1.0
    a = port.Csr.from_any(m)
    lam = float(__import__("scipy.sparse.linalg", fromlist=["eigsh"]).eigsh(m, k=1, which="LA", v0=np.ones(n))[0][0])
    return a.scaled(1.0 / lam)


def test_diag_cluster_tables_bitwise(mc):
    """Q_c wider than one CTA's shared table is held by a cluster of 2/4/8 CTAs
    in distributed shared memory (k_diag_qc): the estimate equals the
    global-table path (MCF_DIAG_CLUSTER=0) bit for bit, for every cluster cap,
    also when the columns' tables are handed to the GPU-wide k_diag_big."""
    import os
    a = _multi_hub_graph()
    g = mc.DeviceGraph(as_matrix(a, True))
    cfg = mc.WalkConfig(a.n * 120, 1e-300, 20, 5)
    outs = {}
    os.environ["MCF_DIAG_UNITS"] = "0"
    try:
        for k in ("0", "2", "4", "8"):
            # BIG_WORK 4096: most hub columns handed to k_diag_big; LONG_WORK 16:
            # hundreds of (i, c) entries split into shared ranges, in groups
            for big, long_ in ((None, None), ("4096", None), (None, "16")):
                os.environ["MCF_DIAG_CLUSTER"] = k
                for var, val in (("MCF_DIAG_BIG_WORK", big), ("MCF_DIAG_LONG_WORK", long_),
                                 ("MCF_DIAG_LONG_WORK_Q", long_)):
                    if val:
                        os.environ[var] = val
                    else:
                        os.environ.pop(var, None)
                outs[k, big, long_] = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values
    finally:
        os.environ.pop("MCF_DIAG_CLUSTER", None)
        os.environ.pop("MCF_DIAG_BIG_WORK", None)
        os.environ.pop("MCF_DIAG_LONG_WORK", None)
        os.environ.pop("MCF_DIAG_LONG_WORK_Q", None)
        os.environ.pop("MCF_DIAG_UNITS", None)
    # the default combine (units: tables split by key group, every probe local)
    # with its natural splits, with every column split into up to 128 units,
    # and with tiny pieces of the queued entries
    try:
        for need, chunk, part in ((None, None, None), ("64", None, None), ("700", "32", None), ("64", None, "0")):
            for var, val in (("MCF_UNIT_SMALL_NEED", need), ("MCF_UNIT_CHUNK", chunk), ("MCF_UNIT_PARTITION", part)):
                if val:
                    os.environ[var] = val
                else:
                    os.environ.pop(var, None)
            outs["units", need, chunk, part] = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values
    finally:
        os.environ.pop("MCF_UNIT_SMALL_NEED", None)
        os.environ.pop("MCF_UNIT_CHUNK", None)
        os.environ.pop("MCF_UNIT_PARTITION", None)
    ref = outs["0", None, None]
    for key, v in outs.items():
        assert np.array_equal(v, ref), key
    assert np.all(np.isfinite(ref)) and np.all(ref > 1.0)


def test_unit_combine_directed_long_column(mc, monkeypatch):
    """An unsymmetric uniform-value graph above the dense-Q size whose column
    0 (20,000 entries) is far longer than any row: the unit combine (default,
    and with every column split) equals the single-table combine bit for bit
    -- CSC-side slices, hub bitmaps from the CSC, an entry queue sized by the
    longest column."""
    rng = np.random.default_rng(7)
    n = 30000
    u, v = rng.integers(0, n, 8 * n), rng.integers(0, n, 8 * n)
    u = np.concatenate([u, rng.choice(np.arange(1, n), 20000, replace=False)])
    v = np.concatenate([v, np.zeros(20000, dtype=np.int64)])
    keep = u != v
    m = sparse.csr_array((np.ones(keep.sum()), (u[keep], v[keep])), shape=(n, n))
    m.sum_duplicates()
    m.data[:] = 1.0
    a = port.Csr.from_any(m)
    assert np.diff(a.csc_ptr).max() > 10 * np.diff(a.row_ptr).max()
    a = a.scaled(1.0 / float(np.diff(a.row_ptr).max()))
    g = mc.DeviceGraph(as_matrix(a, False))
    cfg = mc.WalkConfig(n * 40, 1e-300, 12, 3)
    monkeypatch.setenv("MCF_DIAG_UNITS", "0")
    ref = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values
    monkeypatch.delenv("MCF_DIAG_UNITS")
    out = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values
    assert np.array_equal(out, ref)
    monkeypatch.setenv("MCF_UNIT_SMALL_NEED", "64")
    out = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg).values
    assert np.array_equal(out, ref)
    assert np.all(np.isfinite(ref)) and np.all(ref >= 1.0)


def test_unit_combine_variable_length_walks(mc, monkeypatch):
    """Cutoff-terminated walks (resolvent, max_steps 10^3 > 64: count pass,
    scan, emissions at explicit offsets) through the unit combine, natural
    and forced splits, equal the single-table combine bit for bit."""
    a = _multi_hub_graph(seed=3)
    g = mc.DeviceGraph(as_matrix(a, True))
    cfg = mc.WalkConfig(a.n * 30, 1e-6, 1000, 9)
    monkeypatch.setenv("MCF_DIAG_UNITS", "0")
    ref = mc.rand_funm_diag(g, mc.RESOLVENT, cfg)
    monkeypatch.delenv("MCF_DIAG_UNITS")
    assert ref.emissions > a.n * 30 * 3
    for env in ({}, {"MCF_UNIT_SMALL_NEED": "256"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out = mc.rand_funm_diag(g, mc.RESOLVENT, cfg)
        for k in env:
            monkeypatch.delenv(k)
        assert out.emissions == ref.emissions
        assert np.array_equal(out.values, ref.values), env


def test_rand_funm_full_consistency_and_closed_form(mc):
    """SPEC acceptance 4: diag(rand_funm) == rand_funm_diag (shared seed) to
    1e-12 relative on 16-node instances; SPEC.md:352 closed form; A = 0."""
    rng = np.random.default_rng(1)
    for trial in range(3):
        d = (rng.random((16, 16)) < 0.3).astype(float)
        d = np.triu(d, 1)
        d = d + d.T
        a = mc.SparseMatrix.from_dense(d * 0.2, True)
        cfg = mc.WalkConfig(20_000, 1e-10, 60, trial)
        full = mc.rand_funm(a, mc.EXPONENTIAL, cfg, block=5).values
        diag = mc.rand_funm_diag(a, mc.EXPONENTIAL, cfg).values
        np.testing.assert_allclose(np.diag(full), diag, rtol=1e-12)
        exact = port.dense_funm(port.Csr.from_dense(d * 0.2), "exponential", 64)
        assert np.max(np.abs(full - exact)) < 5e-2
    a2 = mc.SparseMatrix.from_dense([[0, 0.1], [0.1, 0]], True)
    f2 = mc.rand_funm(a2, mc.EXPONENTIAL, mc.WalkConfig(10**6, 1e-10, 10_000, 0)).values
    np.testing.assert_allclose(f2, [[np.cosh(0.1), np.sinh(0.1)], [np.sinh(0.1), np.cosh(0.1)]], atol=5e-3)
    z = mc.rand_funm(mc.SparseMatrix(sparse.csr_array((3, 3)), sparse.csc_array((3, 3))), mc.EXPONENTIAL,
                     mc.WalkConfig(10)).values
    assert np.array_equal(z, np.eye(3))


def test_rand_funm_sparse_products_match_dense(mc):
    """rand_funm's sparse-A block products (mcf_funm_full) equal the dense
    formula z0 I + z1 A + A (Q A) built from the same Q rows (mcf_walk_qdense)
    to rounding, on a weighted non-symmetric 300-node matrix."""
    import torch
    from paper_2308_01037_b200.device import WalkParams
    rng = np.random.default_rng(5)
    n = 300
    m = sparse.random(n, n, density=0.03, random_state=7, format="csr") * 0.3
    m.setdiag(0)
    m.eliminate_zeros()
    m.sort_indices()
    a = mc.SparseMatrix(sparse.csr_array(m), sparse.csc_array(m.tocsc()))
    cfg = mc.WalkConfig(60 * n, 1e-8, 60, 3)
    full = mc.rand_funm(a, mc.EXPONENTIAL, cfg, block=64, as_tensor=True).values
    g = mc.DeviceGraph(a)
    z = mc.EXPONENTIAL.prefix(62)
    ni, pre = g.allocate(cfg.n_walks)
    Q = torch.empty((n, n), dtype=torch.float64, device="cuda")
    g.walk_qdense(WalkParams(cfg, z), pre, Q, (0, n), stats=g.new_stats())
    A = torch.from_numpy(m.toarray()).cuda()
    ref = z[0] * torch.eye(n, dtype=torch.float64, device="cuda") + z[1] * A + A @ (Q @ A)
    assert torch.allclose(full, ref, rtol=1e-12, atol=1e-15)


def test_mc_baseline_full(mc):
    """mc_baseline mode "full": the 2-node path closed form
    (SPEC example: N_s = 1e6 per row within 1e-2 of cosh / sinh 0.1), A = 0 ->
    zeta_0 I, and diag(full) = the MC diagonal of the same walks to 1e-12."""
    a2 = mc.SparseMatrix.from_dense([[0, 0.1], [0.1, 0]], True)
    f2 = mc.mc_baseline(a2, mc.EXPONENTIAL, mc.WalkConfig(10**6, 1e-10, 200, 0), mode="full").values
    np.testing.assert_allclose(f2, [[np.cosh(0.1), np.sinh(0.1)], [np.sinh(0.1), np.cosh(0.1)]], atol=1e-2)
    z = mc.mc_baseline(mc.SparseMatrix(sparse.csr_array((3, 3)), sparse.csc_array((3, 3))), mc.EXPONENTIAL,
                       mc.WalkConfig(10), mode="full").values
    assert np.array_equal(z, np.eye(3))
    c = golden_io.load("er300")
    a = as_matrix(c.sa, True)
    cfg = mc.WalkConfig(200, 1e-8, 40, 4)
    full = mc.mc_baseline(a, mc.EXPONENTIAL, cfg, mode="full").values
    diag = mc.mc_baseline(a, mc.EXPONENTIAL, cfg, mode="diag").values
    np.testing.assert_allclose(np.diag(full), diag, rtol=1e-12, atol=1e-300)
    exact = port.dense_funm(c.sa, "exponential", 40)
    assert np.max(np.abs(full - exact)) < 0.1 * np.max(np.abs(exact))


@pytest.mark.parametrize("uniform", [False, True])
def test_spmv_short_rows_match_sequential_csr_bitwise(mc, uniform):
    """Rows of <= 64 entries: y = z0 v + z1 r + A x equals numpy/scipy's
    sequential CSR evaluation bit for bit (products and sums rounded
    separately, in CSR order) -- the reference computes r = A @ v and
    y = z[0] * v + z[1] * r + A @ q with exactly these operations."""
    import torch
    rng = np.random.default_rng(11)
    n = 5000
    lens = rng.integers(0, 65, n)
    lens[::97] = 64
    lens[::101] = 0
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([rng.choice(n, k, replace=False) for k in lens])
    vals = np.full(rows.size, 0.37) if uniform else rng.normal(size=rows.size)
    m = sparse.csr_array((vals, (rows, cols)), shape=(n, n))
    m.sort_indices()
    a = port.Csr.from_any(m)
    g = mc.DeviceGraph(as_matrix(a))
    x, v, r = rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)
    t = lambda z: torch.from_numpy(z).cuda()  # noqa: E731
    y = g.spmv(t(x)).cpu().numpy()
    assert np.array_equal(y, m @ x)
    y = g.spmv(t(x), alpha=0.75, v=t(v), beta=-1.25, r=t(r)).cpu().numpy()
    assert np.array_equal(y, 0.75 * v + -1.25 * r + m @ x)


@pytest.mark.parametrize("name", ["ba400", "signed6"])
def test_action_v_ones_row_sums(mc, alloc_path, name):
    """v = None (v = 1): r is the reference's A @ ones bit for bit (row sums,
    signed rows summed with their signs), and the estimate equals the one with
    an explicit ones vector (same walks; y to rounding of the hub-row sums)."""
    import torch
    c = golden_io.load(name)
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric))
    cfg = mc.WalkConfig(20 * c.n, 1e-6, 28, 3)
    a1 = mc.rand_funm_action(g, mc.EXPONENTIAL, None, cfg)
    a2 = mc.rand_funm_action(g, mc.EXPONENTIAL, torch.ones(c.n, dtype=torch.float64, device="cuda"), cfg)
    m = sparse.csr_array((c.sa.vals, c.sa.col_ids, c.sa.row_ptr), shape=(c.n, c.n))
    assert np.array_equal(a1.aux["r"].cpu().numpy(), m @ np.ones(c.n))
    np.testing.assert_allclose(a1.values, a2.values, rtol=1e-13, atol=0)
    assert a1.emissions == a2.emissions


def test_device_col_norm_beyond_leaf_cap(mc):
    """A column longer than a warp's leaf table (1024 leaves of <= 128 terms):
    the lane-0 fallback keeps numpy's pairwise bits."""
    rng = np.random.default_rng(5)
    n, deg = 150_001, 140_000
    nb = rng.choice(np.arange(1, n), deg, replace=False)
    rows = np.r_[np.zeros(deg, dtype=np.int64), nb]
    cols = np.r_[nb, np.zeros(deg, dtype=np.int64)]
    m = sparse.coo_array((rng.normal(size=2 * deg), (rows, cols)), shape=(n, n)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    a = port.Csr.from_any(m)
    t = port.transition_tables(a)
    g = mc.DeviceGraph(as_matrix(a))
    d = {k: v.cpu().numpy() for k, v in g.tables().items()}
    assert np.array_equal(d["col_norms"], t.col_norms)
    assert np.array_equal(d["row_abs_sum"], t.rsum)


@pytest.fixture(params=["4", "8"])
def lean_bytes(request):
    """Both lean entry formats: 4-B packed (nnz < 2^25, degree < 63 inline) and 8-B."""
    import os
    os.environ["MCF_LEAN4"] = "1" if request.param == "4" else "0"
    yield request.param
    os.environ.pop("MCF_LEAN4", None)


@pytest.mark.parametrize("name", ["ba400", "er300", "kron8"])
def test_lean_walk_bitwise(mc, lean_bytes, name):
    """v = 1 on a uniform-value graph walks {start, degree} entries with the
    row sums by degree (one dependent load per step): q and y are bitwise the
    ones of the header walk (MCF_LEAN_WALK=0), fat and compact layouts."""
    import os
    import torch
    c = golden_io.load(name)
    a = as_matrix(c.sa, c.symmetric)
    out = {}
    for lean in ("1", "0"):
        os.environ["MCF_LEAN_WALK"] = lean
        try:
            for layout in ("compact", "fat"):
                os.environ["MCF_WALK_LAYOUT"] = layout
                g = mc.DeviceGraph(a, gamma=0.05)
                res = mc.rand_funm_action(g, mc.EXPONENTIAL, None, mc.WalkConfig(30 * c.n, 1e-6, 28, 7))
                out[lean, layout] = (np.asarray(res.values), res.aux["q"].cpu().numpy(), res.emissions)
        finally:
            os.environ.pop("MCF_LEAN_WALK", None)
            os.environ.pop("MCF_WALK_LAYOUT", None)
    ref = out["0", "compact"]
    for k, v in out.items():
        assert np.array_equal(v[0], ref[0]) and np.array_equal(v[1], ref[1]) and v[2] == ref[2], k


@pytest.mark.parametrize("name", ["ba400", "er300", "kron8"])
def test_lean_diag_bitwise(mc, lean_bytes, name):
    """Diag walks on a uniform-value graph use the {start, degree} entries
    with the id read alongside: d is bitwise the header walk's (both layouts)."""
    import os
    c = golden_io.load(name)
    a = as_matrix(c.sa, c.symmetric)
    out = {}
    for lean in ("1", "0"):
        os.environ["MCF_LEAN_WALK"] = lean
        try:
            for layout in ("compact", "fat"):
                os.environ["MCF_WALK_LAYOUT"] = layout
                # lean walks: the one-load {start, id, degree} entries (default)
                # and the lean entry with ecol[e] alongside (MCF_LEAN_ID=0)
                for lid in (("1", "0") if lean == "1" else ("1",)):
                    os.environ["MCF_LEAN_ID"] = lid
                    g = mc.DeviceGraph(a, gamma=0.05)
                    res = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(30 * c.n, 1e-6, 28, 7))
                    out[lean, layout, lid] = (np.asarray(res.values), res.emissions, res.truncated)
        finally:
            os.environ.pop("MCF_LEAN_WALK", None)
            os.environ.pop("MCF_WALK_LAYOUT", None)
            os.environ.pop("MCF_LEAN_ID", None)
    ref = out["0", "compact", "1"]
    for k, v in out.items():
        assert np.array_equal(v[0], ref[0]) and v[1:] == ref[1:], k


def test_lean_walk_absorbing_and_self_loops(mc, lean_bytes):
    """Uniform-value directed graph with sink rows (absorbing) and self loops:
    the lean walk (action v = 1 and diag) matches the header walk bitwise."""
    import os
    rng = np.random.default_rng(3)
    n = 500
    rows = rng.integers(0, n, 3000)
    cols = rng.integers(0, n, 3000)
    keep = rows % 7 != 0                     # every 7th row is a sink
    rows, cols = np.r_[rows[keep], np.arange(0, n, 11)], np.r_[cols[keep], np.arange(0, n, 11)]  # + self loops
    m = sparse.coo_array((np.full(rows.size, 0.3), (rows, cols)), shape=(n, n)).tocsr()
    m.sum_duplicates()
    m.data[:] = 0.3
    m.sort_indices()
    a = as_matrix(port.Csr.from_any(m))
    out = {}
    for lean in ("1", "0"):
        os.environ["MCF_LEAN_WALK"] = lean
        try:
            g = mc.DeviceGraph(a, gamma=0.5)
            cfg = mc.WalkConfig(20 * n, 1e-6, 40, 9)
            ya = mc.rand_funm_action(g, mc.EXPONENTIAL, None, cfg)
            yd = mc.rand_funm_diag(g, mc.EXPONENTIAL, cfg)
            out[lean] = (np.asarray(ya.values), ya.emissions, ya.absorbed, np.asarray(yd.values), yd.emissions)
        finally:
            os.environ.pop("MCF_LEAN_WALK", None)
    assert out["1"][2] > 0  # some walks were absorbed
    for x, y in zip(out["1"], out["0"]):
        assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.parametrize("n_walks", [1, 7, 333])
def test_funm_action_sparse_budgets(mc, alloc_path, n_walks):
    """Budgets far below n (most columns without walks): the one-call action
    (budgets, walks, y) equals the step-by-step path (mcf_allocate_walks,
    mcf_walk_action, mcf_spmv) bit for bit, and the walks number n_walks."""
    import torch
    c = golden_io.load("ba400")
    g = mc.DeviceGraph(as_matrix(c.sa, c.symmetric), gamma=0.05)
    cfg = mc.WalkConfig(n_walks, 1e-6, 28, 5)
    ones = torch.ones(c.n, dtype=torch.float64, device="cuda")
    one_call = mc.rand_funm_action(g, mc.EXPONENTIAL, ones, cfg)
    ni, _ = g.allocate(n_walks)
    stepwise = mc.rand_funm_action(g, mc.EXPONENTIAL, ones, cfg, budgets=ni.cpu().numpy())
    assert one_call.walks == n_walks == stepwise.walks
    assert np.array_equal(np.asarray(one_call.values), np.asarray(stepwise.values))
