"""CPU oracle: a numpy restatement of the reference walk-sampling estimator.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this module;
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may use it, and only as the checker or
as the timed CPU baseline -- never as the thing measured or shipped.

Parity status: PINNED.  ``tests/golden/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/mcfunm``, importable only in the build container) and
stores its transition tables, walk budgets, recorded entry streams and
estimates under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
port against them bit for bit.  The reference ships no estimator module
(SURVEY.md §0), so the estimator layer below restates SPEC.md:358-377 /
PAPER.md Alg. 2, Eq. 20 and Alg. 3 on top of the restated walker; the golden
script performs the same accumulation on top of the *reference* walker.

Third-party arithmetic this follows (same as the reference): numpy 2.3.5's
PCG64DXSM + SeedSequence for the per-column streams (walker.py:173-180),
``np.searchsorted`` on the global ``cdf_key`` (walker.py:281), ``np.cumsum`` and
``np.add.at`` (walker.py:114, sparsemat.py:359), scipy's CSC minor-axis
``reduceat`` for column norms (walker.py:127).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy import sparse

ABSORBING = -1  # walker.py:41


# --------------------------------------------------------------------------
# graph container used by the oracle (plain arrays, no product types)
# --------------------------------------------------------------------------
@dataclass
class Csr:
    """Square sparse matrix as CSR + CSC arrays (cf. sparsemat.py:29-100)."""

    n: int
    row_ptr: np.ndarray   # int64 [n+1]
    col_ids: np.ndarray   # int64 [nnz]
    vals: np.ndarray      # f64   [nnz]
    csc_ptr: np.ndarray = None
    csc_rows: np.ndarray = None
    csc_vals: np.ndarray = None

    def __post_init__(self):
        self.row_ptr = np.asarray(self.row_ptr, dtype=np.int64)
        self.col_ids = np.asarray(self.col_ids, dtype=np.int64)
        self.vals = np.asarray(self.vals, dtype=np.float64)
        if self.csc_ptr is None:
            m = self.scipy_csr().tocsc()
            m.sort_indices()
            self.csc_ptr = m.indptr.astype(np.int64)
            self.csc_rows = m.indices.astype(np.int64)
            self.csc_vals = m.data.astype(np.float64)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def scipy_csr(self):
        return sparse.csr_array((self.vals, self.col_ids, self.row_ptr), shape=(self.n, self.n))

    def scipy_csc(self):
        return sparse.csc_array((self.csc_vals, self.csc_rows, self.csc_ptr), shape=(self.n, self.n))

    def diagonal(self) -> np.ndarray:
        return self.scipy_csr().diagonal()

    def scaled(self, gamma: float) -> "Csr":
        """sparsemat.py:338-352 -- every stored value times gamma."""
        return Csr(self.n, self.row_ptr, self.col_ids, self.vals * gamma,
                   self.csc_ptr, self.csc_rows, self.csc_vals * gamma)

    @classmethod
    def from_any(cls, a) -> "Csr":
        """Accepts a reference/product SparseMatrix (``.csr``/``.csc``) or a scipy matrix."""
        if hasattr(a, "csr") and hasattr(a, "csc"):
            r, c = a.csr, a.csc
        else:
            r = sparse.csr_array(a)
            r.sort_indices()
            c = r.tocsc()
            c.sort_indices()
        return cls(r.shape[0], r.indptr, r.indices, r.data, c.indptr, c.indices, c.data)

    @classmethod
    def from_dense(cls, d) -> "Csr":
        d = np.asarray(d, dtype=np.float64)
        m = sparse.csr_array(d)
        m.sort_indices()
        return cls.from_any(m)


# --------------------------------------------------------------------------
# transition tables (walker.py:97-145) and budgets (walker.py:148-170)
# --------------------------------------------------------------------------
def row_abs_sums(a: Csr) -> np.ndarray:
    """Sequential per-row |a| sums in CSR order (sparsemat.py:355-360)."""
    out = np.zeros(a.n)
    if a.nnz:
        rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_ptr))
        np.add.at(out, rows, np.abs(a.vals))
    return out


@dataclass
class Tables:
    n: int
    row_ptr: np.ndarray
    col_ids: np.ndarray
    row_cdf: np.ndarray
    cdf_key: np.ndarray
    step_ratio: np.ndarray
    rsum: np.ndarray
    col_norms: np.ndarray
    init_prob: np.ndarray


def transition_tables(a: Csr) -> Tables:
    """Restates build_transition_model (walker.py:97-145).

    * within-row CDF from a *global* running sum of |a| (walker.py:113-117),
      last entry of every non-empty row pinned to 1 (walker.py:120-121);
    * global search key row + cdf (walker.py:122);
    * weight update a/t = copysign(row |a| sum, a) (walker.py:124-125);
    * start distribution p_j = ||C_j||_2 / sum ||C||_2 (walker.py:127-129),
      the column sums of squares reduced per CSC column like scipy's
      minor-axis ``reduceat``.
    """
    if a.nnz == 0:
        raise ValueError("degenerate: all columns are zero")  # walker.py:100-103
    rsum = row_abs_sums(a)
    deg = np.diff(a.row_ptr)
    row_of = np.repeat(np.arange(a.n, dtype=np.int64), deg)
    mag = np.abs(a.vals)
    run = np.cumsum(mag)
    base = np.concatenate([[0.0], run])[a.row_ptr[row_of]]
    cdf = np.minimum((run - base) / rsum[row_of], 1.0)
    cdf[a.row_ptr[1:][deg > 0] - 1] = 1.0
    key = row_of + cdf
    ratio = np.copysign(rsum[row_of], a.vals)

    sq = a.csc_vals * a.csc_vals
    cdeg = np.diff(a.csc_ptr)
    nz_cols = np.flatnonzero(cdeg)
    colsq = np.zeros(a.n)
    colsq[nz_cols] = np.add.reduceat(sq, a.csc_ptr[nz_cols])
    norms = np.sqrt(colsq)
    p = norms / norms.sum()
    return Tables(a.n, a.row_ptr, a.col_ids, cdf, key, ratio, rsum, norms, p)


def largest_remainder(p: np.ndarray, total: int) -> np.ndarray:
    """walker.py:148-162: floor(p*N) plus one for the largest remainders,
    ties broken by ascending index (stable sort), p == 0 never gets a walk."""
    p = np.asarray(p, dtype=np.float64)
    want = p * total
    got = np.floor(want).astype(np.int64)
    left = int(total - got.sum())
    if left > 0:
        rem = want - got
        rem[p == 0.0] = -1.0
        got[np.argsort(-rem, kind="stable")[:left]] += 1
    return got


def allocate(t: Tables, n_walks: int) -> np.ndarray:
    """walker.py:165-170."""
    if n_walks < 1:
        raise ValueError("n_walks must be at least 1")
    return largest_remainder(t.init_prob, int(n_walks))


def column_stream(seed: int, column: int) -> np.random.Generator:
    """walker.py:173-180: PCG64DXSM keyed by SeedSequence(seed, spawn_key=(c,))."""
    return np.random.Generator(np.random.PCG64DXSM(np.random.SeedSequence(entropy=seed, spawn_key=(column,))))


# --------------------------------------------------------------------------
# walk drivers
# --------------------------------------------------------------------------
def batch_walks(t: Tables, start: int, n_walks: int, max_steps: int, cutoff: float,
                rng, on_step, on_draw=None):
    """Synchronised walks from one column (walker.py:245-290).

    on_step(k, states, weights, ids) sees the live walks before the absorbing
    filter; on_draw(k, ids, entries) (oracle extension, used to record the
    sampled index stream for replay) sees the walks that drew at step k and the
    CSR entries they took.  Returns (emissions, truncated).
    """
    w0 = 1.0 / n_walks
    thr = cutoff * w0
    states = np.full(n_walks, start, dtype=np.int64)
    weights = np.full(n_walks, w0)
    ids = np.arange(n_walks)
    emitted = 0
    k = 0
    while states.size and k < max_steps:
        on_step(k, states, weights, ids)
        emitted += states.size
        live = t.row_ptr[states + 1] > t.row_ptr[states]
        if not live.all():
            states, weights, ids = states[live], weights[live], ids[live]
            if not states.size:
                return emitted, 0
        u = rng.random(states.size)
        e = np.searchsorted(t.cdf_key, states + u, side="right")
        if on_draw is not None:
            on_draw(k, ids, e)
        weights = weights * t.step_ratio[e]
        states = t.col_ids[e]
        k += 1
        keep = np.abs(weights) > thr
        if not keep.all():
            states, weights, ids = states[keep], weights[keep], ids[keep]
    return emitted, (int(states.size) if k >= max_steps else 0)


def _coeff(tag: str, k: int) -> float:
    """series.py:52-60 -- 1/k! by repeated division, or 1 for the resolvent."""
    if tag == "resolvent":
        return 1.0
    x = 1.0
    for i in range(1, k + 1):
        x /= i
    return x


def _ratio(tag: str, k: int) -> float:
    """series.py:62-67 -- zeta_{k+1}/zeta_k."""
    return 1.0 if tag == "resolvent" else 1.0 / (k + 1)


def single_walk(t: Tables, tag: str, start: int, max_steps: int, cutoff: float, sink,
                w0: float = 1.0, rng=None, seed: int = 0):
    """Scalar walk (walker.py:205-242): per-row inverse-CDF draw (:183-189),
    emits (k, state, zeta_{k+2} W) while |W| > cutoff |w0| and k < max_steps.
    Returns (emissions, truncated)."""
    if rng is None:
        rng = column_stream(seed, start)
    state, w, thr, k = int(start), float(w0), cutoff * abs(w0), 0
    z = _coeff(tag, 2)
    while abs(w) > thr:
        if k >= max_steps:
            return k, True
        sink(k, state, z * w)
        lo, hi = t.row_ptr[state], t.row_ptr[state + 1]
        if lo == hi:
            return k + 1, False
        e = int(lo + np.searchsorted(t.row_cdf[lo:hi], rng.random(), side="right"))
        w *= t.step_ratio[e]
        state = int(t.col_ids[e])
        z *= _ratio(tag, k + 2)
        k += 1
    return k, False


# --------------------------------------------------------------------------
# estimators (Alg. 2 / Eq. 20 / Alg. 3)
# --------------------------------------------------------------------------
def zeta_prefix(tag: str, count: int) -> np.ndarray:
    """series.py:69-80 -- exponential 1/k! by cumulative product, resolvent 1."""
    if count <= 0:
        return np.empty(0)
    if tag == "resolvent":
        return np.ones(count)
    z = np.empty(count)
    z[0] = 1.0
    if count > 1:
        with np.errstate(under="ignore"):
            z[1:] = np.cumprod(1.0 / np.arange(1.0, count))
    return z


@dataclass
class Record:
    """Recorded entry stream in per-walk layout: walk g = walk_pre[c] + w takes
    entries[walk_off[g]:walk_off[g+1]] in step order."""

    walk_pre: np.ndarray
    walk_off: np.ndarray
    entries: np.ndarray


@dataclass
class Run:
    payload: np.ndarray
    ni: np.ndarray
    emissions: int = 0
    truncated: int = 0
    walks: int = 0
    aux: dict = field(default_factory=dict)
    record: Record | None = None


class _Recorder:
    def __init__(self, ni: np.ndarray):
        self.walk_pre = np.concatenate([[0], np.cumsum(ni)]).astype(np.int64)
        self.steps = []  # (global walk ids, entries)

    def hook(self, c):
        base = self.walk_pre[c]

        def on_draw(k, ids, e):
            self.steps.append((base + ids, e.copy()))
        return on_draw

    def finish(self) -> Record:
        total = int(self.walk_pre[-1])
        cnt = np.zeros(total, dtype=np.int64)
        for g, _ in self.steps:
            cnt[g] += 1
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        ent = np.zeros(int(off[-1]), dtype=np.int64)
        fill = off[:-1].copy()
        for g, e in self.steps:  # steps of one column arrive in k order
            ent[fill[g]] = e
            fill[g] += 1
        return Record(self.walk_pre, off, ent)


def funm_action(a: Csr, tag: str, v: np.ndarray, n_walks: int, cutoff: float = 1e-6,
                max_steps: int = 10_000, seed: int = 0, record: bool = False,
                columns=None, per_walk: bool = False) -> Run:
    """RandFunmAction.

    r = A v; q_c = sum_walks sum_k zeta_{k+2} W_k r[l_k] with W_0 = 1/N_c;
    y = zeta_0 v + zeta_1 r + A q.  ``columns`` restricts the walked columns
    (a sample, for the CPU baseline); then y is only partially meaningful.
    """
    v = np.asarray(v, dtype=np.float64)
    z = zeta_prefix(tag, max_steps + 2)
    if a.nnz == 0:  # no walk possible, H-term only
        return Run(z[0] * v, np.zeros(a.n, dtype=np.int64))
    t = transition_tables(a)
    ni = allocate(t, n_walks)
    A = a.scipy_csr()
    r = A @ v
    q = np.zeros(a.n)
    rec = _Recorder(ni) if record else None
    xw = np.zeros(int(ni.sum())) if per_walk else None
    wpre = np.concatenate([[0], np.cumsum(ni)])
    em = tr = 0
    cols = np.flatnonzero(ni) if columns is None else [c for c in columns if ni[c] > 0]
    for c in cols:
        acc = [0.0]
        base = wpre[c]

        def on_step(k, s, w, ids, acc=acc, base=base):
            contrib = w * r[s]
            acc[0] += z[k + 2] * contrib.sum()
            if xw is not None:
                xw[base + ids] += z[k + 2] * contrib
        e, tt = batch_walks(t, int(c), int(ni[c]), max_steps, cutoff, column_stream(seed, int(c)),
                            on_step, rec.hook(c) if rec else None)
        q[c] = acc[0]
        em += e
        tr += tt
    y = z[0] * v + z[1] * r + A @ q
    out = Run(y, ni, em, tr, int(ni[cols].sum()) if len(cols) else 0, {"q": q, "r": r})
    if xw is not None:
        out.aux["x_walk"] = xw
    if rec:
        out.record = rec.finish()
    return out


def funm_diag(a: Csr, tag: str, n_walks: int, cutoff: float = 1e-6, max_steps: int = 10_000,
              seed: int = 0, record: bool = False, columns=None) -> Run:
    """RandFunmDiag.

    Q_c[j] = sum over visits of j by walks from c of zeta_{k+2} W_k (W_0 = 1/N_c);
    Eq. 20: d_i = zeta_0 + zeta_1 a_ii + sum_c a_ic <Q_c, C_i>, one Q row live
    at a time.
    """
    z = zeta_prefix(tag, max_steps + 2)
    if a.nnz == 0:
        return Run(np.full(a.n, z[0]), np.zeros(a.n, dtype=np.int64))
    t = transition_tables(a)
    ni = allocate(t, n_walks)
    d = z[0] + z[1] * a.diagonal()
    rec = _Recorder(ni) if record else None
    em = tr = 0
    qrow = np.zeros(a.n)
    cols = np.flatnonzero(ni) if columns is None else [c for c in columns if ni[c] > 0]
    for c in cols:
        qrow[:] = 0.0

        def on_step(k, s, w, ids):
            np.add.at(qrow, s, z[k + 2] * w)
        e, tt = batch_walks(t, int(c), int(ni[c]), max_steps, cutoff, column_stream(seed, int(c)),
                            on_step, rec.hook(c) if rec else None)
        em += e
        tr += tt
        lo, hi = a.csc_ptr[c], a.csc_ptr[c + 1]
        for i, aic in zip(a.csc_rows[lo:hi], a.csc_vals[lo:hi]):
            ilo, ihi = a.csc_ptr[i], a.csc_ptr[i + 1]
            d[i] += aic * (qrow[a.csc_rows[ilo:ihi]] @ a.csc_vals[ilo:ihi])
    out = Run(d, ni, em, tr, int(ni[cols].sum()) if len(cols) else 0)
    if rec:
        out.record = rec.finish()
    return out


# --------------------------------------------------------------------------
# replay of a recorded entry stream (what the device replay kernels must match)
# --------------------------------------------------------------------------
def replay(a: Csr, tag: str, rec: Record, max_steps: int, cutoff: float, mode: str,
           v: np.ndarray | None = None) -> np.ndarray:
    """Re-walks every recorded walk from its entry list (pure Python; small
    cases only) and accumulates like funm_action / funm_diag.  Used to prove
    that a recorded stream fully determines the estimate."""
    t = transition_tables(a)
    z = zeta_prefix(tag, max_steps + 2)
    n = a.n
    ni = np.diff(rec.walk_pre)
    A = a.scipy_csr()
    if mode == "action":
        r = A @ np.asarray(v, dtype=np.float64)
        q = np.zeros(n)
    else:
        d = z[0] + z[1] * a.diagonal()
    for c in np.flatnonzero(ni):
        w0 = 1.0 / ni[c]
        thr = cutoff * w0
        qrow = np.zeros(n) if mode == "diag" else None
        for g in range(rec.walk_pre[c], rec.walk_pre[c + 1]):
            ents = rec.entries[rec.walk_off[g]:rec.walk_off[g + 1]]
            s, w, k, j = int(c), w0, 0, 0
            while k < max_steps:
                if mode == "action":
                    q[c] += z[k + 2] * w * r[s]
                else:
                    qrow[s] += z[k + 2] * w
                if t.row_ptr[s + 1] == t.row_ptr[s]:
                    break
                e = int(ents[j])
                j += 1
                w *= t.step_ratio[e]
                s = int(t.col_ids[e])
                k += 1
                if not abs(w) > thr:
                    break
            assert j == len(ents), "recorded stream and walk termination disagree"
        if mode == "diag":
            lo, hi = a.csc_ptr[c], a.csc_ptr[c + 1]
            for i, aic in zip(a.csc_rows[lo:hi], a.csc_vals[lo:hi]):
                ilo, ihi = a.csc_ptr[i], a.csc_ptr[i + 1]
                d[i] += aic * (qrow[a.csc_rows[ilo:ihi]] @ a.csc_vals[ilo:ihi])
    if mode == "action":
        return z[0] * v + z[1] * r + A @ q
    return d


# --------------------------------------------------------------------------
# exact references (oracle.py:42-136) and extras
# --------------------------------------------------------------------------
def dense_funm(a: Csr, tag: str, terms: int) -> np.ndarray:
    """oracle.py:42-80: sum_{k<=terms} zeta_k A^k by dense powers (n <= 2048)."""
    if a.n > 2048:
        raise ValueError("dense evaluation capped at n=2048")
    ad = a.scipy_csr().toarray()
    z = zeta_prefix(tag, terms + 1)
    out = z[0] * np.eye(a.n)
    p = np.eye(a.n)
    for k in range(1, terms + 1):
        p = p @ ad
        if z[k] != 0.0:
            out += z[k] * p
    return out


def taylor_action(a: Csr, tag: str, v: np.ndarray, terms: int) -> np.ndarray:
    """sum_{k<=terms} zeta_k A^k v by the SpMV recurrence (exact action oracle)."""
    A = a.scipy_csr()
    z = zeta_prefix(tag, terms + 1)
    x = np.asarray(v, dtype=np.float64).copy()
    out = z[0] * x
    for k in range(1, terms + 1):
        x = A @ x
        out += z[k] * x
    return out


def q_exact(a: Csr, tag: str, v: np.ndarray, max_steps: int) -> np.ndarray:
    """E[q] = sum_{k<max_steps} zeta_{k+2} A^{k+1} v (per walked column)."""
    A = a.scipy_csr()
    z = zeta_prefix(tag, max_steps + 2)
    x = A @ np.asarray(v, dtype=np.float64)
    out = np.zeros(a.n)
    for k in range(max_steps):
        out += z[k + 2] * x
        x = A @ x
    return out


def expm_diag_eigh(a: Csr) -> np.ndarray:
    """diag(exp(A)) for symmetric A via a dense eigendecomposition."""
    w, U = np.linalg.eigh(a.scipy_csr().toarray())
    return (U * U) @ np.exp(w)


def cg_solve(a: Csr, gamma: float, b: np.ndarray, tol: float = 1e-10, max_iter: int = 1000):
    """oracle.py:83-125: unpreconditioned CG on (I - gamma A) x = b."""
    A = a.scipy_csr()
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rs = float(r @ r)
    lim = tol * np.linalg.norm(b)
    if np.sqrt(rs) <= lim:
        return x
    for _ in range(max_iter):
        ap = p - gamma * (A @ p)
        al = rs / float(p @ ap)
        x += al * p
        r -= al * ap
        rn = float(r @ r)
        if np.sqrt(rn) <= lim:
            return x
        p = r + (rn / rs) * p
        rs = rn
    raise RuntimeError("cg did not converge")


def gershgorin_gamma(a: Csr, fraction: float) -> float:
    """oracle.py:128-136."""
    return fraction / float(np.max(row_abs_sums(a)))


# --------------------------------------------------------------------------
# column-sample drivers for the CPU baseline (bench.py cpu_baseline and
# --impl reference legs): the same per-column loop as funm_action /
# funm_diag, restricted to a set of start columns.
# --------------------------------------------------------------------------
def action_columns(t: Tables, r: np.ndarray, z: np.ndarray, ni: np.ndarray, cols, max_steps: int,
                   cutoff: float, seed: int):
    """q_c for the given columns (dict) and the emissions they made."""
    out, em = {}, 0
    for c in cols:
        acc = [0.0]

        def on_step(k, s, w, ids, acc=acc):
            acc[0] += z[k + 2] * (w * r[s]).sum()
        e, _ = batch_walks(t, int(c), int(ni[c]), max_steps, cutoff, column_stream(seed, int(c)), on_step)
        out[int(c)] = acc[0]
        em += e
    return out, em


def _ranges(starts: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Concatenation of the index ranges [starts[k], starts[k] + lens[k])."""
    tot = int(lens.sum())
    if tot == 0:
        return np.zeros(0, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)[:-1]])
    return np.repeat(starts - off, lens) + np.arange(tot, dtype=np.int64)


def diag_columns(a: Csr, t: Tables, z: np.ndarray, ni: np.ndarray, cols, max_steps: int, cutoff: float,
                 seed: int, out: np.ndarray | None = None, chunk_ids: int = 1 << 22):
    """Eq. 20 contributions of the given columns and their emissions: the
    reference walker (batch_walks = walker.py:245-290) builds Q_c as in
    funm_diag, then d_i += a_ic <Q_c, C_i> for i in C_c, the inner products
    vectorised over all of C_c (gather of the C_i row ids, products, segment
    sums; at most ``chunk_ids`` ids at a time).  Q_c is reset only where the
    walks touched it.  Returns ({i: sum}, emissions), or (out, emissions) when
    a dense accumulator ``out`` is given."""
    contrib, em = ({} if out is None else out), 0
    qrow = np.zeros(a.n)
    for c in cols:
        touched = []

        def on_step(k, s, w, ids):
            np.add.at(qrow, s, z[k + 2] * w)
            touched.append(s)
        e, _ = batch_walks(t, int(c), int(ni[c]), max_steps, cutoff, column_stream(seed, int(c)), on_step)
        em += e
        lo, hi = a.csc_ptr[c], a.csc_ptr[c + 1]
        rows, aic = a.csc_rows[lo:hi], a.csc_vals[lo:hi]
        starts, lens = a.csc_ptr[rows], a.csc_ptr[rows + 1] - a.csc_ptr[rows]
        p = 0
        while p < rows.size:  # groups of C_c entries with at most chunk_ids ids in total
            q = p + max(1, int(np.searchsorted(np.cumsum(lens[p:]), chunk_ids, side="right")))
            idx = _ranges(starts[p:q], lens[p:q])
            prod = qrow[a.csc_rows[idx]] * a.csc_vals[idx]
            seg = np.zeros(q - p)
            nz = lens[p:q] > 0
            if idx.size:
                bounds = np.concatenate([[0], np.cumsum(lens[p:q])[:-1]])[nz]
                seg[nz] = np.add.reduceat(prod, bounds)
            vals = aic[p:q] * seg
            if out is None:
                for i, v in zip(rows[p:q], vals):
                    contrib[int(i)] = contrib.get(int(i), 0.0) + v
            else:
                np.add.at(out, rows[p:q], vals)
            p = q
        if touched:
            qrow[np.concatenate(touched)] = 0.0
    return contrib, em


# --------------------------------------------------------------------------
# single-entry estimator and the classic MC baseline (SPEC-only in the
# reference: Alg. 1 :93-117 and §4.3 :636-649)
# --------------------------------------------------------------------------
def entry_budgets(t: Tables, a: Csr, i: int, n_walks: int) -> np.ndarray:
    """walks only from the columns j with a_ij != 0, the start
    distribution renormalised over that support, largest-remainder rounding."""
    lo, hi = a.row_ptr[i], a.row_ptr[i + 1]
    cols = a.col_ids[lo:hi]
    ni = np.zeros(a.n, dtype=np.int64)
    if hi > lo:
        p = t.init_prob[cols]
        if p.sum() > 0:
            ni[cols] = largest_remainder(p / p.sum(), n_walks)
    return ni


def funm_entry(a: Csr, tag: str, v: np.ndarray, i: int, n_walks: int, cutoff: float = 1e-6,
               max_steps: int = 10_000, seed: int = 0, record: bool = False) -> Run:
    """y_i = zeta_0 v_i + zeta_1 r_i + <A_i, q> with q from walks launched only
    from row i's support."""
    v = np.asarray(v, dtype=np.float64)
    z = zeta_prefix(tag, max_steps + 2)
    lo, hi = a.row_ptr[i], a.row_ptr[i + 1]
    if hi == lo:  # empty row: zeta_0 v_i exactly, no walk
        return Run(np.array([z[0] * v[i]]), np.zeros(a.n, dtype=np.int64))
    t = transition_tables(a)
    ni = entry_budgets(t, a, i, n_walks)
    A = a.scipy_csr()
    r = A @ v
    rec = _Recorder(ni) if record else None
    q = np.zeros(a.n)
    em = tr = 0
    for c in np.flatnonzero(ni):
        acc = [0.0]

        def on_step(k, s, w, ids, acc=acc):
            acc[0] += z[k + 2] * (w * r[s]).sum()
        e, tt = batch_walks(t, int(c), int(ni[c]), max_steps, cutoff, column_stream(seed, int(c)), on_step,
                            rec.hook(c) if rec else None)
        q[c] = acc[0]
        em += e
        tr += tt
    yi = z[0] * v[i] + z[1] * r[i] + a.vals[lo:hi] @ q[a.col_ids[lo:hi]]
    out = Run(np.array([yi]), ni, em, tr, int(ni.sum()), {"q": q, "r": r})
    if rec:
        out.record = rec.finish()
    return out


def mc_baseline(a: Csr, tag: str, walks_per_row: int, cutoff: float = 1e-6, max_steps: int = 10_000,
                seed: int = 0, mode: str = "diag", v: np.ndarray | None = None, rows=None,
                record: bool = False) -> Run:
    """Alg. 1: N_s walks from every row i, W0 = 1/N_s,
    f_{i,l_k} += zeta_k W_k.  diag keeps f_ii (walks back at i); action
    accumulates y_i += zeta_k W_k v[l_k]; ``rows`` restricts the start rows
    (entry mode).  Walks use the same per-row substreams and batch driver."""
    z = zeta_prefix(tag, max_steps + 1)
    t = transition_tables(a)
    rows = np.arange(a.n) if rows is None else np.asarray(rows)
    ni = np.zeros(a.n, dtype=np.int64)
    ni[rows] = walks_per_row
    rec = _Recorder(ni) if record else None
    out = np.zeros(a.n)
    if mode == "action":
        v = np.asarray(v, dtype=np.float64)
    em = tr = 0
    for i in rows:
        acc = [0.0]

        def on_step(k, s, w, ids, acc=acc, i=int(i)):
            if mode == "action":
                acc[0] += z[k] * (w * v[s]).sum()
            else:
                acc[0] += z[k] * w[s == i].sum()
        e, tt = batch_walks(t, int(i), int(walks_per_row), max_steps, cutoff, column_stream(seed, int(i)), on_step,
                            rec.hook(i) if rec else None)
        out[i] = acc[0]
        em += e
        tr += tt
    res = Run(out, ni, em, tr, int(ni.sum()))
    if rec:
        res.record = rec.finish()
    return res


# --------------------------------------------------------------------------
# node-subset replay at full size ("for large configs, replay a
# node subset S using columns U_{a in S} N(a)")
# --------------------------------------------------------------------------
def record_subset(a: Csr, t: Tables, z: np.ndarray, ni: np.ndarray, cols, subset, max_steps: int,
                  cutoff: float, seed: int):
    """Walk the given columns with the reference walker (batch_walks,
    per-column PCG64DXSM streams) over the FULL model, recording every walk's
    entry stream, and accumulate the Eq. 20 terms of the nodes in ``subset``
    only: d_a += a_ac <Q_c, C_a> for a in subset and C_c.  Returns
    ([(c, walk_off_local int64[N_c + 1], entries int32)], {a: sum}, emissions)."""
    sub = set(int(x) for x in subset)
    recs, contrib, em = [], {}, 0
    qrow = np.zeros(a.n)
    for c in cols:
        c = int(c)
        nc = int(ni[c])
        steps = []
        touched = []

        def on_step(k, s, w, ids):
            np.add.at(qrow, s, z[k + 2] * w)
            touched.append(s)

        def on_draw(k, ids, e):
            steps.append((ids.copy(), e.astype(np.int32)))
        e_, _ = batch_walks(t, c, nc, max_steps, cutoff, column_stream(seed, c), on_step, on_draw)
        em += e_
        cnt = np.zeros(nc, dtype=np.int64)
        for ids, _ in steps:
            cnt[ids] += 1
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        ent = np.empty(int(off[-1]), dtype=np.int32)
        fill = off[:-1].copy()
        for ids, e in steps:  # steps arrive in k order: per-walk streams stay in step order
            ent[fill[ids]] = e
            fill[ids] += 1
        recs.append((c, off, ent))
        lo, hi = a.csc_ptr[c], a.csc_ptr[c + 1]
        for i, aic in zip(a.csc_rows[lo:hi], a.csc_vals[lo:hi]):
            if int(i) in sub:
                ilo, ihi = a.csc_ptr[i], a.csc_ptr[i + 1]
                contrib[int(i)] = contrib.get(int(i), 0.0) + aic * (qrow[a.csc_rows[ilo:ihi]] @ a.csc_vals[ilo:ihi])
        if touched:
            qrow[np.concatenate(touched)] = 0.0
    return recs, contrib, em
