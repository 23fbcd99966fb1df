"""Parity on the BASELINE configurations themselves (device RNG, full size).

* config 1 (ER n=1e4 LCC, diag): every node's estimate against the exact
  diagonal of exp(beta A) (fp64 eigh on the GPU), with the per-node standard
  error of rand_funm_diag(stderr=True);
* config 2 (BA n=1e6, action): the reference's entry streams for every
  walked column replayed at full size (1e-10);
* config 3 (R-MAT 2^22, diag): the multi-batch emission path and the
  big-column fallback give the same d bit for bit as the default batching.

Acceptance (the multiplicity-controlled form of "every node within
3 sigma"): |z| <= 3 for >= 99% of nodes, max |z| within the Bonferroni bound
for n nodes at family-wise level 0.01, z mean ~ 0 and sd ~ 1.
Graphs come from the bench recipe (tools/bench_graphs.py)."""
import math
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import bench  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _z_acceptance(z, dof=None, what="", mean_tol=0.05):
    from scipy import stats
    n = z.size
    alpha = 0.01 / (2 * n)
    bound = stats.t.ppf(1 - alpha, dof) if dof else stats.norm.ppf(1 - alpha)
    frac3 = float(np.mean(np.abs(z) <= 3))
    msg = (f"{what}: n={n} frac|z|<=3 {frac3:.5f} max|z| {np.max(np.abs(z)):.3f} (bound {bound:.3f}) "
           f"mean {z.mean():.4f} sd {z.std():.4f}")
    print(msg)
    sd_ref = math.sqrt(dof / (dof - 2)) if dof else 1.0
    assert frac3 >= 0.99, msg
    assert np.max(np.abs(z)) <= bound, msg
    assert abs(z.mean()) < mean_tol, msg
    assert abs(z.std() / sd_ref - 1) < 0.08, msg


def _device_graph(cfg):
    import paper_2308_01037_b200 as mc
    a, beta, n_walks = bench.make_graph(cfg)
    return mc.DeviceGraph(a, gamma=beta), beta, n_walks


def test_config1_diag_vs_exact_eigh():
    """Config 1: d = diag exp(beta A) on the ER(1e4) LCC, 1000 walks per node,
    30 Taylor terms (max_steps 28), W_c = 1e-300; SE from 16 walk groups."""
    _need_gpu()
    import paper_2308_01037_b200 as mc
    cfg = bench.CONFIGS[1]
    g, beta, n_walks = _device_graph(cfg)
    res = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], 11),
                            stderr=True, groups=16)
    A = torch.zeros((g.n, g.n), dtype=torch.float64, device="cuda")
    rows = torch.repeat_interleave(torch.arange(g.n, device="cuda"), g.row_ptr.diff())
    A[rows, g.col_ids.to(torch.int64)] = g.vals
    lam, V = torch.linalg.eigh(A)
    exact = ((V * V) @ torch.exp(lam)).cpu().numpy()  # 30-term Taylor = expm to ~1e-16 at beta lambda_max = 1
    assert res.stderr is not None and np.all(res.stderr > 0)
    z = (res.values - exact) / res.stderr
    _z_acceptance(z, what="config1 diag")
    rel = np.abs(res.values - exact) / exact
    assert np.max(rel) < 1e-3  # ~1e-4 single run


_WREC = {}


def _weighted_worker(cols):
    from oracle import port
    s = _WREC
    recs, _, em = port.record_subset(s["A"], s["t"], s["z"], s["ni"], cols, [], s["max_steps"], s["cutoff"],
                                     s["seed"])
    q, _ = port.action_columns(s["t"], s["r"], s["z"], s["ni"], cols, s["max_steps"], s["cutoff"], s["seed"])
    return recs, q, em


def _record_action(A, t, ni, z, r, max_steps, cutoff, seed):
    """Entry streams of every walked column by the reference walker (oracle
    port, forked pool over column chunks) and the reference's q; returns the
    replay Record, y = z0 + z1 r + A q (v = 1) and the emission count."""
    import multiprocessing as mp

    from oracle import port
    _WREC.update(A=A, t=t, z=z, ni=ni, r=r, max_steps=max_steps, cutoff=cutoff, seed=seed)
    cols = np.flatnonzero(ni)
    procs = os.cpu_count() or 1
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_weighted_worker, [c for c in np.array_split(cols, procs * 8) if c.size])
    n = A.n
    q = np.zeros(n)
    recs = []
    em = 0
    for rr, qq, e in parts:
        recs += rr
        em += e
        for c, v in qq.items():
            q[c] = v
    y_ref = z[0] + z[1] * r + A.scipy_csr() @ q
    walk_pre = np.concatenate([[0], np.cumsum(ni)])
    walk_off = np.zeros(int(walk_pre[-1]) + 1, dtype=np.int64)
    ents, base = [], 0
    for c, off, ent in sorted(recs, key=lambda x: x[0]):
        g0 = walk_pre[c]
        walk_off[g0 + 1:g0 + off.size] = base + off[1:]
        ents.append(ent)
        base += ent.size
    walk_off = np.maximum.accumulate(walk_off)
    return port.Record(walk_pre, walk_off, np.concatenate(ents)), y_ref, em


def test_config2_full_replay():
    """Config 2 at FULL size (BA n = 1e6, m = 4, 640,000 walks, 30 Taylor
    terms): the reference walker's entry streams for every walked column
    (PCG64DXSM per column, global searchsorted) replayed on the device give the
    reference's exp(beta A) 1 to 1e-10 (north-star replay mode), with the same
    emission count; the device budgets equal the reference allocation.

    (The device-RNG z-test of SURVEY 4 is not applied here: with N_i in
    {0, 1, 2} the per-node estimate at beta lambda_max = 1 is heavy-tailed --
    walks through hubs multiply their weight by beta deg per step -- so the
    replicate mean sits below the masked target with an underestimated spread.
    The reference algorithm itself shows it: 64 replicates of the oracle port
    on BA(2e4) give z mean -0.26, max |z| 14.9 (DESIGN 5).  Config 1 carries
    the statistical check.)"""
    _need_gpu()
    import paper_2308_01037_b200 as mc
    from oracle import port
    cfg = bench.CONFIGS[2]
    a, beta, n_walks = bench.make_graph(cfg)
    n = a.n
    rp = np.asarray(a.csr.indptr, dtype=np.int64)
    ci = np.asarray(a.csr.indices, dtype=np.int64)
    A = port.Csr(n, rp, ci, np.full(ci.size, beta), rp, ci, np.full(ci.size, beta))
    t = port.transition_tables(A)
    ni = port.allocate(t, n_walks)
    z = port.zeta_prefix("exponential", cfg["max_steps"] + 2)
    r = A.scipy_csr() @ np.ones(n)
    rec, y_ref, em = _record_action(A, t, ni, z, r, cfg["max_steps"], cfg["cutoff"], cfg["seed"])
    g = mc.DeviceGraph(a, gamma=beta)
    dni, _ = g.allocate(n_walks)
    assert np.array_equal(dni.cpu().numpy(), ni)
    res = mc.rand_funm_action(g, mc.EXPONENTIAL, np.ones(n), mc.WalkConfig(n_walks, cfg["cutoff"],
                                                                           cfg["max_steps"], cfg["seed"]), replay=rec)
    rel = np.max(np.abs(res.values - y_ref) / np.abs(y_ref))
    print(f"config2 full replay: walks {n_walks} emissions {em} max rel err {rel:.3e}")
    assert res.emissions == em
    assert rel < 1e-10


def test_config3_multibatch_and_pool_fallback_bitwise(monkeypatch):
    """Config 3 at full size: the default combine (units), the single-table /
    cluster / GPU-wide combine it replaced (MCF_DIAG_UNITS=0), 4x more emission
    batches (MCF_EMISSION_SLOTS = 2^28), serial and overlapped batches
    (MCF_DIAG_OVERLAP) and, on the old combine, no big-column pool
    (MCF_DIAG_POOL=0: the allocation-failure path) give the same d bit for bit."""
    _need_gpu()
    import paper_2308_01037_b200 as mc
    cfg = bench.CONFIGS[3]
    g, beta, n_walks = _device_graph(cfg)
    wc = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], 0)
    ref = mc.rand_funm_diag(g, mc.EXPONENTIAL, wc, as_tensor=True)
    assert ref.emissions > 1.8e10
    # (MCF_DIAG_OVERLAP: serial batches / the next batch's walk beside the combine on 8 or 24 reserved SMs)
    for env in ({"MCF_EMISSION_SLOTS": str(1 << 28)}, {"MCF_UNIT_PARTITION": "0"}, {"MCF_DIAG_OVERLAP": "0"},
                {"MCF_DIAG_OVERLAP": "8"}, {"MCF_DIAG_OVERLAP": "24", "MCF_EMISSION_SLOTS": str(1 << 28)},
                {"MCF_DIAG_UNITS": "0"}, {"MCF_DIAG_UNITS": "0", "MCF_DIAG_POOL": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out = mc.rand_funm_diag(g, mc.EXPONENTIAL, wc, as_tensor=True)
        for k in env:
            monkeypatch.delenv(k)
        assert out.emissions == ref.emissions
        assert torch.equal(out.values, ref.values), env


_SUB = {}


def _subset_worker(cols):
    from oracle import port
    s = _SUB
    return port.record_subset(s["A"], s["t"], s["z"], s["ni"], cols, s["S"], s["max_steps"], s["cutoff"],
                              s["seed"])


def test_config3_node_subset_replay():
    """Config 3 (R-MAT 2^22, 200 walks/node, 23 steps) at FULL size: the
    reference walker (oracle port, PCG64DXSM streams, global searchsorted over
    the 1.3e8-entry cdf_key) walks every column adjacent to a degree-
    stratified node subset S over the full model, its entry streams drive the
    device walks (replay), and d_a for a in S must agree to 1e-10 (SURVEY
    8(c)).  The device runs its full-size tables, budgets and combine paths;
    the subset's columns include the top hubs (node 0, degree ~1.6e5, is
    adjacent to most of S), whose Q_c go through the wide-table paths.  The
    walk budgets are checked bitwise against the reference allocation at the
    full config as well."""
    _need_gpu()
    import multiprocessing as mp

    import paper_2308_01037_b200 as mc
    from oracle import port
    cfg = bench.CONFIGS[3]
    a, beta, n_walks = bench.make_graph(cfg)
    g = mc.DeviceGraph(a, gamma=beta)
    n = a.n
    rp = np.asarray(a.csr.indptr, dtype=np.int64)
    ci = np.asarray(a.csr.indices, dtype=np.int64)
    vals = np.full(ci.size, beta)
    A = port.Csr(n, rp, ci, vals, rp, ci, vals)
    t = port.transition_tables(A)
    ni = port.allocate(t, n_walks)
    dni, _ = g.allocate(n_walks)
    assert np.array_equal(dni.cpu().numpy(), ni), "walk budgets differ from the reference allocation"
    deg = np.diff(rp)
    # S: 4 nodes per degree octave [2^k, 2^(k+1)) up to 2^11, the walks of
    # their neighbourhoods capped so the CPU oracle finishes in about a minute
    rng = np.random.default_rng(7)
    S = []
    for k in range(12):
        cand = np.flatnonzero((deg >= 1 << k) & (deg < 2 << k))
        rng.shuffle(cand)
        took = 0
        for v in cand[:400]:
            w = ni[ci[rp[v]:rp[v + 1]]].sum()
            if w <= 400_000:
                S.append(int(v))
                took += 1
            if took == 4:
                break
    # and low-degree neighbours of the four top hubs: the hub columns
    # themselves (widest Q_c: cluster / global-table / GPU-wide paths) are walked
    for h in np.argsort(-deg, kind="stable")[:4]:
        nb = ci[rp[h]:rp[h + 1]]
        nb = nb[deg[nb] <= 8]
        S += [int(v) for v in rng.choice(nb, size=min(2, nb.size), replace=False)]
    S = np.array(sorted(set(S)))
    cols = np.unique(np.concatenate([ci[rp[v]:rp[v + 1]] for v in S]))
    cols = cols[ni[cols] > 0]
    assert 0 in cols.tolist(), "the top hub should be among the walked columns"
    z = port.zeta_prefix("exponential", cfg["max_steps"] + 2)
    _SUB.update(A=A, t=t, z=z, ni=ni, S=S, max_steps=cfg["max_steps"], cutoff=cfg["cutoff"], seed=cfg["seed"])
    procs = os.cpu_count() or 1
    chunks = [c for c in np.array_split(cols, procs * 4) if c.size]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_subset_worker, chunks)
    recs = sorted((r for p in parts for r in p[0]), key=lambda r: r[0])
    d_ref = np.full(S.size, z[0])  # no self loops: a_aa = 0
    for p in parts:
        for v, x in p[1].items():
            d_ref[np.searchsorted(S, v)] += x
    # the recorded streams in the per-walk layout of the replay API
    ni_s = np.zeros(n, dtype=np.int64)
    ni_s[cols] = ni[cols]
    walk_pre = np.concatenate([[0], np.cumsum(ni_s)])
    walk_off = np.zeros(int(walk_pre[-1]) + 1, dtype=np.int64)
    ents = []
    base = 0
    for c, off, ent in recs:
        g0 = walk_pre[c]
        walk_off[g0 + 1:g0 + off.size] = base + off[1:]
        ents.append(ent)
        base += ent.size
    # columns in walk order are ascending, so walk_off is monotone after a fill-forward
    walk_off = np.maximum.accumulate(walk_off)
    rec = port.Record(walk_pre, walk_off, np.concatenate(ents))
    res = mc.rand_funm_diag(g, mc.EXPONENTIAL, mc.WalkConfig(int(walk_pre[-1]), cfg["cutoff"], cfg["max_steps"],
                                                             cfg["seed"]), replay=rec)
    em = sum(p[2] for p in parts)
    assert res.emissions == em
    rel = np.abs(res.values[S] - d_ref) / np.abs(d_ref)
    print(f"config3 subset replay: |S|={S.size} columns={cols.size} walks={walk_pre[-1]} emissions={em} "
          f"max rel err {rel.max():.3e}")
    assert rel.max() < 1e-10


def test_weighted_signed_replay_1e5():
    """Weighted, signed rows at 1e5 nodes (the inverse-CDF
    draw and the copysign(row sum, a) weight update, walker.py:112-125):
    the reference walker's entry streams on the weighted Barabasi-Albert graph
    (n = 1e5, |w| ~ U[0.5, 1.5), 10% negative) replayed on the device give
    the reference's f(A) 1 to 1e-10; the device-RNG estimate (alias-table
    draws) agrees with the exact series by the SURVEY 4 rule (per-walk SEs)."""
    _need_gpu()
    import paper_2308_01037_b200 as mc
    from oracle import port
    from paper_2308_01037_b200.sparsemat import SparseMatrix
    from tools import bench_graphs
    gd = bench_graphs.load({"graph": "ba_signed", "n": 100_000, "m": 4, "seed": 3})
    n, rp, ci, w = gd["n"], gd["row_ptr"], gd["col_ids"], gd["vals"]
    gamma = 1.0 / gd["lambda_max"]
    a = SparseMatrix.from_csr_arrays(n, rp, ci, w, symmetric_hint=True)
    A = port.Csr(n, rp, ci.astype(np.int64), w * gamma, rp, ci.astype(np.int64), w * gamma)
    t = port.transition_tables(A)
    max_steps, cutoff, seed, n_walks = 28, 1e-300, 5, 4 * n
    ni = port.allocate(t, n_walks)
    z = port.zeta_prefix("exponential", max_steps + 2)
    r = A.scipy_csr() @ np.ones(n)
    rec, y_ref, em = _record_action(A, t, ni, z, r, max_steps, cutoff, seed)
    g = mc.DeviceGraph(a, gamma=gamma)
    assert g.info["n_uniform_rows"] < n // 2  # weighted: the non-uniform (alias / CDF) paths
    cfg = mc.WalkConfig(n_walks, cutoff, max_steps, seed)
    res = mc.rand_funm_action(g, mc.EXPONENTIAL, np.ones(n), cfg, replay=rec)
    rel = np.max(np.abs(res.values - y_ref) / np.maximum(np.abs(y_ref), 1e-300))
    print(f"weighted replay n={n}: emissions {em} max rel err {rel:.3e}")
    assert res.emissions == em
    assert rel < 1e-10
    # device RNG against the exact 30-term series, per-walk SEs: alias-table
    # draws (default) and the inverse-CDF search (MCF_ALIAS=0) must both pass
    # the rule and agree with each other (same walks' law, different draws).
    # The z mean is allowed 0.1 here: at beta rho = 1 on a BA graph the per-walk
    # weights are heavy-tailed (hub rows multiply them by beta sum |w|), which
    # pulls the z distribution slightly negative for any implementation.
    exact = port.taylor_action(A, "exponential", np.ones(n), max_steps + 1)
    means = {}
    for alias in ("1", "0"):
        os.environ["MCF_ALIAS"] = alias
        try:
            ga = mc.DeviceGraph(a, gamma=gamma)
            est = mc.rand_funm_action(ga, mc.EXPONENTIAL, np.ones(n), mc.WalkConfig(400 * n, cutoff, max_steps, 9),
                                      stderr=True)
        finally:
            os.environ.pop("MCF_ALIAS", None)
        ok = est.stderr > 0
        zsc = (est.values[ok] - exact[ok]) / est.stderr[ok]
        means[alias] = float(zsc.mean())
        _z_acceptance(zsc, what=f"weighted device RNG (alias={alias})", mean_tol=0.1)
    assert abs(means["1"] - means["0"]) < 0.03, means
