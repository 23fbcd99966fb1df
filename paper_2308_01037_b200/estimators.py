"""Drop-in estimators: RandFunmDiag and RandFunmAction on the GPU.

Signatures follow the reference SPEC:
    rand_funm_diag(a, coeffs, config)      -> FunmResult (diagonal d)
    rand_funm_action(a, coeffs, v, config) -> FunmResult (vector y)
``a`` is a SparseMatrix-like object already scaled by gamma (reference or this
package's type) or a resident ``DeviceGraph``.  The per-column loop, the walks
and the accumulation all run in libmcfunm_cuda.so kernels.

Two sampling modes:
  * device RNG (default): Philox-4x32-10 keyed by (seed, column, walk, step);
    statistically equivalent to the reference, partition-invariant;
  * replay: ``replay=`` a recorded reference entry stream (walk_pre, walk_off,
    entries, as produced by oracle/ or tests/golden); the device then
    reproduces the reference estimate to summation-order rounding.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .device import DeviceGraph, WalkParams, to_host
from .errors import ArgumentError
from .series import as_stream
from .walker import check_config


@dataclass
class FunmResult:
    """Estimator output: payload plus walk statistics."""

    values: np.ndarray
    kind: str
    walks: int = 0
    emissions: int = 0
    truncated: int = 0
    absorbed: int = 0
    config: dict = field(default_factory=dict)
    stderr: np.ndarray | None = None
    aux: dict = field(default_factory=dict)

    @property
    def payload(self) -> np.ndarray:
        return self.values

    @property
    def mean_steps(self) -> float:
        return self.emissions / self.walks if self.walks else 0.0


def _graph(a, device=None) -> DeviceGraph:
    return a if isinstance(a, DeviceGraph) else DeviceGraph(a, device=device)


def _n_nnz(a):
    if isinstance(a, DeviceGraph):
        return a.n, a.nnz
    return int(a.csr.shape[0]), int(a.csr.nnz)


def _cfg_echo(cfg, coeffs, mode):
    return {"n_walks": cfg.n_walks, "weight_cutoff": cfg.weight_cutoff, "max_steps": cfg.max_steps,
            "seed": cfg.seed, "function": coeffs.tag, "sampling": mode}


def _budgets(g: DeviceGraph, cfg, replay, budgets):
    """(ni, walk_pre, total walks).  Explicit budgets and replay streams carry
    their own walk count, which becomes the calls' exact walk_capacity (the
    device buffers are sized by it; a mismatch with config.n_walks is fine)."""
    if replay is not None:
        pre = np.asarray(replay.walk_pre, dtype=np.int64)
        if pre.size != g.n + 1:
            raise ArgumentError("replay stream has the wrong number of columns")
        ni = np.diff(pre)
        return (*g.budgets(ni), int(ni.sum()))
    if budgets is not None:
        b = np.asarray(budgets, dtype=np.int64)
        return (*g.budgets(b), int(b.sum()))
    return (*g.allocate(cfg.n_walks), int(cfg.n_walks))


def _replay_tensors(g: DeviceGraph, replay):
    off = torch.from_numpy(np.ascontiguousarray(replay.walk_off, dtype=np.int64)).to(g.device)
    ent = np.asarray(replay.entries)
    if ent.size and (ent.min() < 0 or ent.max() >= g.nnz):
        raise ArgumentError("replay entries outside [0, nnz)")
    ent = torch.from_numpy(np.ascontiguousarray(ent, dtype=np.int32)).to(g.device)
    return off, ent


def _stats(res: FunmResult, st: torch.Tensor):
    s = st.cpu().numpy()
    res.walks, res.emissions, res.truncated, res.absorbed = (int(x) for x in s[:4])


def rand_funm_action(a, coeffs, v, config, *, replay=None, budgets=None, stderr: bool = False,
                     device=None, as_tensor: bool = False) -> FunmResult:
    """y ~ f(A) v = zeta_0 v + zeta_1 A v + A q  (Alg. 3).

    r = A v; q_c = sum over the N_c walks from column c of
    sum_k zeta_{k+2} W_k r[l_k] with W_0 = 1/N_c; y = zeta_0 v + zeta_1 r + A q.
    ``v=None`` means v = 1 (total communicability, Katz): r is then the row
    sums of A, bit-identical to A @ ones, without a SpMV.
    """
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    ones = v is None
    v_np = np.ones(n) if ones else (None if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64))
    if (v.shape if isinstance(v, torch.Tensor) else v_np.shape) != (n,):
        raise ArgumentError(f"v must have length {n}")
    z = coeffs.prefix(cfg.max_steps + 2)
    mode = "replay" if replay is not None else "philox"
    if nnz == 0:  # no walk can start: H-term only
        vals = (z[0] * (v_np if v_np is not None else v.cpu().numpy()))
        return FunmResult(vals, "action", config=_cfg_echo(cfg, coeffs, mode))
    g = _graph(a, device)
    vd = v.to(g.device, torch.float64) if isinstance(v, torch.Tensor) else torch.from_numpy(v_np).to(g.device)
    params = WalkParams(cfg, z, g.device)
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    qvar = torch.zeros_like(q) if stderr else None
    st = g.new_stats()
    if replay is None and budgets is None:
        # budgets, r = A v, walks, q, y = z0 v + z1 r + A q in one library call
        r = torch.empty_like(q)
        y, ni, pre = g.funm_action(params, cfg.n_walks, None if ones else vd, z[0], z[1], r, q, torch.empty_like(q),
                                   qvar, st)
    elif replay is None:
        ni, pre, total = _budgets(g, cfg, replay, budgets)
        r = g.spmv(vd)
        g.walk_action(params.derive(capacity=total), pre, r, q, qvar, stats=st)
        y = g.spmv(q, alpha=z[0], v=vd, beta=z[1], r=r)
    else:
        ni, pre, total = _budgets(g, cfg, replay, budgets)
        r = g.spmv(vd)                       # r = A v
        off, ent = _replay_tensors(g, replay)
        g.replay_action(params.derive(capacity=total), pre, off, ent, r, q, stats=st)
        y = g.spmv(q, alpha=z[0], v=vd, beta=z[1], r=r)   # y = z0 v + z1 r + A q
    res = FunmResult(y if as_tensor else to_host(y), "action", config=_cfg_echo(cfg, coeffs, mode))
    _stats(res, st)
    res.aux = {"q": q, "r": r, "ni": ni, "walk_pre": pre}
    if stderr:
        # Var(y_a) = sum_i a_ai^2 Var(q_i): SpMV with squared values
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            a2 = torch.sparse_csr_tensor(g.row_ptr, g.col_ids.to(torch.int64), g.vals * g.vals, (g.n, g.n),
                                         check_invariants=False)
            res.stderr = torch.sqrt(a2 @ qvar).cpu().numpy()
    return res


def rand_funm_diag(a, coeffs, config, *, replay=None, budgets=None, device=None,
                   as_tensor: bool = False, stderr: bool = False, groups: int = 16) -> FunmResult:
    """d ~ diag f(A) by Eq. 20:
    d_i = zeta_0 + zeta_1 a_ii + sum_c a_ic <Q_c, C_i>,
    Q_c[j] = sum over visits of j by walks from c of zeta_{k+2} W_k (W_0 = 1/N_c).

    ``stderr=True`` attaches the Monte Carlo standard error of every d_i
    (SPEC.md:410): ``groups`` more passes, each walking only the walks
    w = g mod groups of every column (same Philox streams), give per-entry
    batch means whose spread estimates Var(pcol[(i, c)]); the columns are
    independent, so Var(d_i) is their sum (mcf_diag_variance).  Device RNG
    only; costs ``groups`` extra estimator passes."""
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    z = coeffs.prefix(cfg.max_steps + 2)
    mode = "replay" if replay is not None else "philox"
    if nnz == 0:  # A = 0 -> d = zeta_0 exactly
        return FunmResult(np.full(n, z[0]), "diag", config=_cfg_echo(cfg, coeffs, mode))
    if stderr and replay is not None:
        raise ArgumentError("stderr needs device-RNG walks (not replay)")
    if stderr and not 2 <= int(groups) <= 256:
        raise ArgumentError("groups must be in [2, 256]")
    g = _graph(a, device)
    ni, pre, total = _budgets(g, cfg, replay, budgets)
    params = WalkParams(cfg, z, g.device).derive(capacity=total)
    pcol = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    if replay is None:
        g.walk_diag(params, pre, pcol, stats=st)
    else:
        off, ent = _replay_tensors(g, replay)
        g.replay_diag(params, pre, off, ent, pcol, stats=st)
    d = g.diag_combine(z[0], z[1], pcol)
    res = FunmResult(d if as_tensor else to_host(d), "diag", config=_cfg_echo(cfg, coeffs, mode))
    _stats(res, st)
    res.aux = {"pcol": pcol, "ni": ni, "walk_pre": pre}
    if stderr:
        from . import _native as N
        G = int(groups)
        pg = torch.zeros((G, g.nnz), dtype=torch.float64, device=g.device)
        gst = g.new_stats()
        for k in range(G):
            g.walk_diag(params.derive(flags=N.group_flags(G, k)), pre, pg[k], stats=gst)
        var = g.diag_variance(pg, pre)
        res.stderr = torch.sqrt(var).cpu().numpy()
        res.aux["groups"] = G
    return res


def _row(g: DeviceGraph, i: int):
    lo, hi = (int(x) for x in g.row_ptr[i:i + 2].cpu())
    return lo, hi, g.col_ids[lo:hi].to(torch.int64), g.vals[lo:hi]


def rand_funm_entry(a, coeffs, v, i: int, config, *, replay=None, device=None) -> FunmResult:
    """(f(A) v)_i alone (§4.3 :636-649):
    y_i = zeta_0 v_i + zeta_1 r_i + <A_i, q>, with walks launched only from the
    columns j where a_ij != 0 and the start distribution renormalised over that
    support (largest-remainder rounding, as allocate_walks)."""
    from .walker import largest_remainder
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    if not 0 <= int(i) < n:
        raise ArgumentError(f"entry index {i} outside [0, {n})")
    v_np = v.cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
    if v_np.shape != (n,):
        raise ArgumentError(f"v must have length {n}")
    z = coeffs.prefix(cfg.max_steps + 2)
    mode = "replay" if replay is not None else "philox"
    empty = FunmResult(np.array([z[0] * v_np[i]]), "entry", config=_cfg_echo(cfg, coeffs, mode))
    if nnz == 0:
        return empty
    g = _graph(a, device)
    lo, hi, cols, vals = _row(g, int(i))
    if hi == lo:  # empty row: y_i = zeta_0 v_i exactly, no walk
        return empty
    if replay is not None:
        ni, pre, total = _budgets(g, cfg, replay, None)
    else:
        p = g.tables()["init_prob"][cols].cpu().numpy()
        nib = np.zeros(n, dtype=np.int64)
        if p.sum() > 0:
            nib[cols.cpu().numpy()] = largest_remainder(p / p.sum(), cfg.n_walks)
        ni, pre = g.budgets(nib)
        total = int(nib.sum())
    vd = torch.from_numpy(np.ascontiguousarray(v_np)).to(g.device)
    params = WalkParams(cfg, z, g.device).derive(capacity=total)
    r = g.spmv(vd)
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    if replay is None:
        g.walk_action(params, pre, r, q, stats=st)
    else:
        off, ent = _replay_tensors(g, replay)
        g.replay_action(params, pre, off, ent, r, q, stats=st)
    yi = float(z[0] * vd[i] + z[1] * r[i] + (vals * q[cols]).sum())
    res = FunmResult(np.array([yi]), "entry", config=_cfg_echo(cfg, coeffs, mode))
    _stats(res, st)
    res.aux = {"q": q, "r": r, "ni": ni}
    return res


def mc_baseline(a, coeffs, config, mode: str = "diag", *, v=None, i: int | None = None, replay=None,
                device=None) -> FunmResult:
    """Classic Monte Carlo (Alg. 1 :93-117) on the same
    device walk engine: ``config.n_walks`` walks from EVERY row (Alg. 1's per-row
    N_s; total n N_s), W0 = 1/N_s, each step adds zeta_k W_k (from k = 0).
    mode "diag": f_ii (only emissions back at i); "action": y_i = sum zeta_k
    W_k v[l_k]; "entry": the action of row i only; "full": the whole n x n
    estimate F[i, j] = sum over the walks from i of zeta_k W_k [l_k = j]
    (dense rows from the walk emissions, mcf_walk_qdense; n <= 16384)."""
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    if mode not in ("diag", "action", "entry", "full"):
        raise ArgumentError(f"mc_baseline mode must be diag, action, entry or full (got '{mode}')")
    n, nnz = _n_nnz(a)
    z = coeffs.prefix(cfg.max_steps + 1)
    zs = np.concatenate([[0.0, 0.0], z])  # the kernel reads zeta[k + 2]: shift Alg. 1's zeta_k by two
    if mode == "full":
        return _mc_full(a, coeffs, cfg, z, zs, n, nnz, device)
    if mode in ("action", "entry"):
        if v is None:
            raise ArgumentError("action/entry mode needs v")
        v_np = v.cpu().numpy() if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
        if v_np.shape != (n,):
            raise ArgumentError(f"v must have length {n}")
    if mode == "entry" and (i is None or not 0 <= int(i) < n):
        raise ArgumentError("entry mode needs a row index i in [0, n)")
    smode = "replay" if replay is not None else "philox"
    if nnz == 0:  # A = 0: f = zeta_0 I
        vals = np.full(n, z[0]) if mode == "diag" else z[0] * v_np
        return FunmResult(vals if mode != "entry" else np.array([vals[i]]), "mc-" + mode,
                          config=_cfg_echo(cfg, coeffs, smode))
    g = _graph(a, device)
    rows = [int(i)] if mode == "entry" else None
    rtotal = None
    if replay is not None:
        ni, pre, rtotal = _budgets(g, cfg, replay, None)
    else:
        nib = np.zeros(n, dtype=np.int64)
        nib[rows if rows is not None else slice(None)] = cfg.n_walks
        ni, pre = g.budgets(nib)
    from . import _native as N
    from .walker import WalkConfig
    pcfg = WalkConfig(max(1, cfg.n_walks * (1 if rows else n)), cfg.weight_cutoff, cfg.max_steps, cfg.seed)
    params = WalkParams(pcfg, zs, g.device)
    payload = (torch.from_numpy(np.ascontiguousarray(v_np)).to(g.device) if mode != "diag"
               else torch.zeros(g.n, dtype=torch.float64, device=g.device))
    if mode == "diag":
        params.c.flags |= N.MCF_FLAG_RETURN_ONLY
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    if replay is None:
        # < 2^31 walks per launch: chunk the start rows
        per = max(1, (1 << 30) // max(1, cfg.n_walks))
        ranges = [(int(i), int(i) + 1)] if rows else [(lo, min(n, lo + per)) for lo in range(0, n, per)]
        for lo, hi in ranges:
            params.c.walk_capacity = cfg.n_walks * (hi - lo)
            g.walk_action(params, pre, payload, q, cols=(lo, hi), stats=st)
    else:
        off, ent = _replay_tensors(g, replay)
        g.replay_action(params.derive(capacity=rtotal), pre, off, ent, payload, q, stats=st)
    out = to_host(q)
    res = FunmResult(out if mode != "entry" else np.array([out[int(i)]]), "mc-" + mode,
                     config=_cfg_echo(cfg, coeffs, smode))
    _stats(res, st)
    return res


def _mc_full(a, coeffs, cfg, z, zs, n, nnz, device, block: int = 1024) -> FunmResult:
    """Alg. 1 full matrix (SPEC.md:389-397 mode "full"): N_s walks from every
    row, W0 = 1/N_s, F[i, l_k] += zeta_k W_k -- the dense Q rows of the walk
    emissions with the coefficient table shifted by two (k_qdense, fixed-point
    accumulation: deterministic)."""
    from .errors import ResourceError
    from .walker import WalkConfig
    if n > 16384:
        raise ResourceError(f"the dense MC estimate needs n <= 16384 (got n={n})")
    if nnz == 0:
        return FunmResult(z[0] * np.eye(n), "mc-full", config=_cfg_echo(cfg, coeffs, "philox"))
    g = _graph(a, device)
    ni, pre = g.budgets(np.full(n, cfg.n_walks, dtype=np.int64))
    params = WalkParams(WalkConfig(max(1, cfg.n_walks * n), cfg.weight_cutoff, cfg.max_steps, cfg.seed), zs, g.device)
    F = torch.empty((n, n), dtype=torch.float64, device=g.device)
    st = g.new_stats()
    per = max(1, min(block, (1 << 30) // max(1, cfg.n_walks)))  # < 2^31 walks per call
    for cb in range(0, n, per):
        ce = min(n, cb + per)
        g.walk_qdense(params.derive(capacity=cfg.n_walks * (ce - cb)), pre, F[cb:ce], (cb, ce), stats=st)
    res = FunmResult(to_host(F), "mc-full", config=_cfg_echo(cfg, coeffs, "philox"))
    _stats(res, st)
    return res


def rand_funm(a, coeffs, config, *, block: int = 1024, device=None, as_tensor: bool = False) -> FunmResult:
    """Full matrix estimate F ~ f(A) = zeta_0 I + zeta_1 A + A Q A (PAPER.md
    Alg. 2 / Eq. 19), Q assembled in row blocks of ``block``
    columns so one block of Q is live at a time.  The walks, the Q rows and the
    two products per block (Q_b A and A[:, block] R, over the SPARSE A) run in
    libmcfunm_cuda (mcf_funm_full).  Dense output: n <= 16384 (ResourceError
    otherwise, advising the diag or action estimators)."""
    from .errors import ResourceError
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    z = coeffs.prefix(cfg.max_steps + 2)
    if n > 16384:
        raise ResourceError(f"the dense estimate needs n <= 16384 (got n={n}): use rand_funm_diag / rand_funm_action")
    if nnz == 0:  # A = 0 -> zeta_0 I exactly
        return FunmResult(z[0] * np.eye(n), "full", config=_cfg_echo(cfg, coeffs, "philox"))
    g = _graph(a, device)
    params = WalkParams(cfg, z, g.device)
    ni, pre = g.allocate(cfg.n_walks)
    F = torch.empty((n, n), dtype=torch.float64, device=g.device)
    st = g.new_stats()
    # blocks of walked columns: Q_b A and A[:, block] (Q_b A) over the sparse A (Eq. 19)
    g.funm_full(params.derive(capacity=0), pre, z[0], z[1], F, block=block, stats=st)
    res = FunmResult(F if as_tensor else to_host(F), "full", config=_cfg_echo(cfg, coeffs, "philox"))
    _stats(res, st)
    res.aux = {"ni": ni, "walk_pre": pre}
    return res
