"""Generate golden fixtures from the REAL reference package.

Run in the build container only (it imports /root/reference/pkg/src/mcfunm,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

For each small graph this records, straight from the reference code:
  * the reference TransitionModel arrays (walker.py:97-145),
  * allocate_walks budgets for several N_s (walker.py:165-170),
  * the sampled entry stream of run_walks_batch (walker.py:245-290), captured by
    wrapping rng_for_column's generator in a logging proxy (SURVEY.md §8c recipe)
    and re-deriving entries = searchsorted(cdf_key, states + u, 'right'),
  * diag / action estimates accumulated on top of the reference walker exactly
    as SPEC.md:358-377 / PAPER.md Alg. 2, Eq. 20, Alg. 3 describe (the
    reference ships no estimator module),
and the SPEC known-answer examples evaluated with the reference functions.
Outputs: tests/golden/<case>.npz and tests/golden/kats.json (reference and
numpy/scipy versions recorded in each file).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import scipy

sys.path.insert(0, "/root/reference/pkg/src")
from mcfunm import graphgen, oracle, series, sparsemat, walker  # noqa: E402
from mcfunm.errors import DegenerateInputError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
VERSIONS = {"numpy": np.__version__, "scipy": scipy.__version__, "reference": "/root/reference@snapshot"}


class LoggingRng:
    """Forwards to the reference generator and keeps every random(size) block."""

    def __init__(self, inner):
        self.inner = inner
        self.blocks = []

    def random(self, size=None):
        x = self.inner.random(size)
        self.blocks.append(np.atleast_1d(np.array(x, copy=True)))
        return x


def walk_column(model, c, n_c, cfg, on_step_acc):
    """Run the reference batch driver for one column and recover its entry stream.

    Returns per-step (ids, entries) for the walks that drew at each step."""
    rng = LoggingRng(walker.rng_for_column(cfg.seed, c))
    seen = []

    def on_step(k, states, weights, ids):
        on_step_acc(k, states, weights, ids)
        seen.append((states.copy(), ids.copy()))

    out = walker.run_walks_batch(model, c, n_c, cfg, rng, on_step)
    steps = []
    for (states, ids), u in zip(seen, rng.blocks):
        live = model.row_ptr[states + 1] > model.row_ptr[states]
        s, i = states[live], ids[live]
        assert s.size == u.size
        steps.append((i, np.searchsorted(model.cdf_key, s + u, side="right")))
    return out, steps


def to_walk_layout(ni, per_col_steps):
    pre = np.concatenate([[0], np.cumsum(ni)]).astype(np.int64)
    cnt = np.zeros(int(pre[-1]), dtype=np.int64)
    for c, steps in per_col_steps.items():
        for ids, _ in steps:
            cnt[pre[c] + ids] += 1
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    ent = np.zeros(int(off[-1]), dtype=np.int64)
    fill = off[:-1].copy()
    for c, steps in per_col_steps.items():
        for ids, e in steps:
            g = pre[c] + ids
            ent[fill[g]] = e
            fill[g] += 1
    return pre, off, ent


def ref_action(a, coeffs, v, cfg):
    model = walker.build_transition_model(a)
    ni = walker.allocate_walks(model, cfg.n_walks)
    z = coeffs.prefix(cfg.max_steps + 2)
    r = a.csr @ v
    q = np.zeros(a.n)
    em = tr = 0
    steps = {}
    for c in np.flatnonzero(ni):
        acc = [0.0]

        def on_step(k, s, w, ids, acc=acc):
            acc[0] += z[k + 2] * (w * r[s]).sum()
        (e, t), st = walk_column(model, int(c), int(ni[c]), cfg, on_step)
        q[c] = acc[0]
        em += e
        tr += t
        steps[int(c)] = st
    y = z[0] * v + z[1] * r + a.csr @ q
    return model, ni, y, q, r, em, tr, to_walk_layout(ni, steps)


def ref_diag(a, coeffs, cfg):
    model = walker.build_transition_model(a)
    ni = walker.allocate_walks(model, cfg.n_walks)
    z = coeffs.prefix(cfg.max_steps + 2)
    d = z[0] + z[1] * a.diagonal()
    qrow = np.zeros(a.n)
    em = tr = 0
    steps = {}
    for c in np.flatnonzero(ni):
        qrow[:] = 0.0

        def on_step(k, s, w, ids):
            np.add.at(qrow, s, z[k + 2] * w)
        (e, t), st = walk_column(model, int(c), int(ni[c]), cfg, on_step)
        em += e
        tr += t
        steps[int(c)] = st
        rows, vals = a.col_entries(int(c))
        for i, aic in zip(rows, vals):
            ri, vi = a.col_entries(int(i))
            d[i] += aic * (qrow[ri] @ vi)
    return d, em, tr, to_walk_layout(ni, steps)


def lam_max(a):
    from scipy.sparse.linalg import eigsh
    if a.n <= 64:
        return float(np.max(np.linalg.eigvalsh(a.toarray())))
    return float(eigsh(a.csr.astype(np.float64), k=1, which="LA")[0][0])


def ba_graph(n, m, seed):
    """Small preferential-attachment graph (fixture input only)."""
    rng = np.random.default_rng(seed)
    edges = [(i, j) for i in range(m + 1) for j in range(i)]
    rep = [x for e in edges for x in e]
    for v in range(m + 1, n):
        t = set()
        while len(t) < m:
            t.add(rep[rng.integers(len(rep))])
        for u in t:
            edges.append((v, u))
            rep += [v, u]
    e = np.array(edges)
    return sparsemat.simple_graph_from_edges(e[:, 0], e[:, 1], directed=False, drop_isolated=False)


def er_lcc(n, deg, seed):
    from scipy.sparse.csgraph import connected_components
    rng = np.random.default_rng(seed)
    m = n * deg // 2
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    g = sparsemat.simple_graph_from_edges(u, v, directed=False, drop_isolated=False)
    _, lab = connected_components(g.csr, directed=False)
    big = np.argmax(np.bincount(lab))
    keep = np.flatnonzero(lab == big)
    sub = g.csr[keep][:, keep].tocoo()
    return sparsemat.SparseMatrix.from_coo(sub.row, sub.col, sub.data, keep.size, symmetric_hint=True)


def cases():
    out = {}
    out["spec3"] = (sparsemat.SparseMatrix.from_dense([[0, 1, 1], [1, 0, 0], [1, 0, 0]], True), 1.0)
    out["inv2"] = (sparsemat.SparseMatrix.from_dense([[0, 1], [1, 0]], True), 0.5)
    # signed, weighted, non-symmetric, with an empty (absorbing) row 4 and a self loop
    dense = np.array([[0, 2, -1, 0, 0, 0.5],
                      [1, 0, 0, 3, 0, 0],
                      [0, -1, 0.25, 0, 1, 0],
                      [0, 0, 1, 0, 0, -2],
                      [0, 0, 0, 0, 0, 0],
                      [1, 0, 0, 1, 1, 0]], dtype=float)
    out["signed6"] = (sparsemat.SparseMatrix.from_dense(dense), 0.2)
    er = er_lcc(300, 8, 0)
    out["er300"] = (er, 1.0 / lam_max(er))
    kr = graphgen.gen_kronecker(graphgen.KroneckerParams(scale=8, edge_factor=16, seed=3))
    out["kron8"] = (kr, 1.0 / lam_max(kr))
    ba = ba_graph(400, 4, 5)
    out["ba400"] = (ba, 1.0 / lam_max(ba))
    sw = graphgen.gen_smallworld(graphgen.SmallWorldParams(n=64, k=4, rewire_prob=0.1, seed=1))
    out["sw64_katz"] = (sw, oracle.gershgorin_gamma(sw, 0.85))
    return out


RUNS = {
    # case: list of (mode, tag, n_walks, cutoff, max_steps, seed)
    "spec3": [("action", "exponential", 3000, 1e-300, 28, 0), ("diag", "exponential", 3000, 1e-300, 28, 0)],
    "inv2": [("action", "exponential", 64, 1e-300, 5, 0), ("diag", "exponential", 64, 1e-300, 5, 1)],
    "signed6": [("action", "exponential", 4000, 1e-6, 40, 2), ("diag", "exponential", 4000, 1e-6, 40, 3),
                ("action", "resolvent", 4000, 1e-8, 200, 4)],
    "er300": [("action", "exponential", 300 * 40, 1e-300, 28, 0), ("diag", "exponential", 300 * 40, 1e-300, 28, 0)],
    "kron8": [("action", "exponential", 20000, 1e-300, 23, 7), ("diag", "exponential", 20000, 1e-300, 23, 7)],
    "ba400": [("action", "exponential", 6400, 1e-300, 28, 11), ("diag", "exponential", 8000, 1e-6, 28, 12)],
    "sw64_katz": [("action", "resolvent", 20000, 1e-8, 10000, 0)],
}


def save_case(name, a, gamma):
    sa = sparsemat.scale(a, gamma)
    model = walker.build_transition_model(sa)
    blob = {
        "n": np.int64(a.n), "gamma": np.float64(gamma),
        "row_ptr": a.csr.indptr.astype(np.int64), "col_ids": a.csr.indices.astype(np.int64),
        "vals": a.csr.data.astype(np.float64),
        "csc_ptr": a.csc.indptr.astype(np.int64), "csc_rows": a.csc.indices.astype(np.int64),
        "csc_vals": a.csc.data.astype(np.float64),
        "symmetric": np.bool_(a.symmetric_hint),
        "m_row_cdf": model.row_cdf, "m_cdf_key": model.cdf_key, "m_step_ratio": model.step_ratio,
        "m_row_abs_sum": model.row_abs_sum, "m_col_norms": model.col_norms, "m_init_prob": model.init_prob,
        "alpha": np.float64(walker.alpha_diagnostic(sa)),
    }
    for ns in (1, 7, 1000, 12345, 10 * a.n + 3):
        blob[f"ni_{ns}"] = walker.allocate_walks(model, ns)
    runs = []
    for j, (mode, tag, nw, cut, ms, seed) in enumerate(RUNS[name]):
        cfg = walker.WalkConfig(n_walks=nw, weight_cutoff=cut, max_steps=ms, seed=seed)
        coeffs = series.CoefficientStream(tag)
        p = f"r{j}_"
        if mode == "action":
            v = np.ones(a.n) if j % 2 == 0 else np.linspace(-1.0, 2.0, a.n)
            _, ni, y, q, r, em, tr, (pre, off, ent) = ref_action(sa, coeffs, v, cfg)
            blob[p + "v"] = v
            blob[p + "y"] = y
            blob[p + "q"] = q
            blob[p + "r"] = r
        else:
            d, em, tr, (pre, off, ent) = ref_diag(sa, coeffs, cfg)
            ni = np.diff(pre)
            blob[p + "d"] = d
        blob[p + "ni"] = ni
        blob[p + "walk_pre"] = pre
        blob[p + "walk_off"] = off
        blob[p + "entries"] = ent.astype(np.int32)
        blob[p + "emissions"] = np.int64(em)
        blob[p + "truncated"] = np.int64(tr)
        runs.append({"mode": mode, "tag": tag, "n_walks": nw, "cutoff": cut, "max_steps": ms, "seed": seed})
    blob["runs_json"] = np.array(json.dumps(runs))
    blob["versions_json"] = np.array(json.dumps(VERSIONS))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **blob)
    print(name, "n", a.n, "nnz", a.nnz, "entries", [int(blob[f'r{j}_entries'].size) for j in range(len(runs))])


def kats():
    k = {"versions": VERSIONS}
    a3 = sparsemat.SparseMatrix.from_dense([[0, 1, 1], [1, 0, 0], [1, 0, 0]])
    m3 = walker.build_transition_model(a3)
    k["spec257_row_cdf"] = m3.row_cdf.tolist()
    k["spec257_col_norms"] = m3.col_norms.tolist()
    k["spec257_init_prob"] = m3.init_prob.tolist()
    k["spec268_alloc"] = walker.allocate_walks(m3, 1000).tolist()
    k["spec269_alloc"] = walker.largest_remainder(np.array([0.9, 0.1]), 1).tolist()
    k["spec267_alloc"] = walker.largest_remainder(np.array([0.5, 0.5]), 10).tolist()
    aw = sparsemat.SparseMatrix.from_dense([[0, 2, -1], [0, 0, 0], [5, 0, 0]])
    mw = walker.build_transition_model(aw)
    k["spec258_step_ratio"] = mw.step_ratio.tolist()
    k["spec80_row_abs_sums"] = sparsemat.row_abs_sums(aw).tolist()
    c4 = sparsemat.SparseMatrix.from_dense(np.roll(np.eye(4), 1, 1) + np.roll(np.eye(4), -1, 1), True)
    k["spec297_alpha"] = walker.alpha_diagnostic(sparsemat.scale(c4, 0.1))
    k["spec466_gershgorin"] = oracle.gershgorin_gamma(c4, 0.85)
    # self loop 0.5, W_c = 0.1 -> 4 emissions, both drivers
    s1 = sparsemat.SparseMatrix.from_dense([[0.5]])
    ms1 = walker.build_transition_model(s1)
    cfg = walker.WalkConfig(n_walks=1, weight_cutoff=0.1, max_steps=100, seed=0)
    em = []
    k["spec287_run_walk"] = list(walker.run_walk(ms1, series.EXPONENTIAL, 0, cfg, lambda *x: em.append(x)))
    k["spec287_batch"] = list(walker.run_walks_batch(ms1, 0, 1, cfg, walker.rng_for_column(0, 0), lambda *x: None))
    # constant weight -> truncated at max_steps
    cw = sparsemat.SparseMatrix.from_dense([[0, 1], [1, 0]])
    mcw = walker.build_transition_model(cw)
    cfg2 = walker.WalkConfig(n_walks=5, weight_cutoff=0.5, max_steps=17, seed=0)
    k["spec288_batch"] = list(walker.run_walks_batch(mcw, 0, 5, cfg2, walker.rng_for_column(0, 0), lambda *x: None))
    k["spec288_run_walk"] = list(walker.run_walk(mcw, series.EXPONENTIAL, 0, cfg2, lambda *x: None))
    k["spec447_cosh"] = oracle.dense_funm(sparsemat.scale(cw, 0.1), series.EXPONENTIAL, 30).values.tolist()
    k["spec448_resolvent"] = oracle.dense_funm(sparsemat.scale(cw, 0.5), series.RESOLVENT, 60).values.tolist()
    k["spec457_cg"] = oracle.cg_solve(cw, 0.5, np.ones(2)).tolist()
    try:
        graphgen.gen_kronecker(graphgen.KroneckerParams(scale=1, edge_factor=1, pa=1.0, pb=0.0, pc=0.0))
        k["spec143_kron_degenerate"] = False
    except DegenerateInputError:
        k["spec143_kron_degenerate"] = True
    k["coeff_exp_0_5"] = [series.EXPONENTIAL.coeff(i) for i in range(6)]
    k["prefix_exp_32"] = series.EXPONENTIAL.prefix(32).tolist()
    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(k, fh, indent=1)


if __name__ == "__main__":
    kats()
    for name, (a, gamma) in cases().items():
        save_case(name, a, gamma)
