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

from .device import DeviceGraph, WalkParams
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
    if replay is not None:
        pre = np.asarray(replay.walk_pre, dtype=np.int64)
        if pre.size != g.n + 1:
            raise ArgumentError("replay stream has the wrong number of columns")
        return g.budgets(np.diff(pre))
    if budgets is not None:
        return g.budgets(budgets)
    return g.allocate(cfg.n_walks)


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
    """
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    v_np = None if isinstance(v, torch.Tensor) else np.asarray(v, dtype=np.float64)
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
    ni, pre = _budgets(g, cfg, replay, budgets)
    r = g.spmv(vd)                       # r = A v
    q = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    qvar = torch.zeros_like(q) if stderr else None
    st = g.new_stats()
    if replay is None:
        g.walk_action(params, pre, r, q, qvar, stats=st)
    else:
        off, ent = _replay_tensors(g, replay)
        g.replay_action(params, pre, off, ent, r, q, stats=st)
    y = g.spmv(q, alpha=z[0], v=vd, beta=z[1], r=r)   # y = z0 v + z1 r + A q
    res = FunmResult(y if as_tensor else y.cpu().numpy(), "action", config=_cfg_echo(cfg, coeffs, mode))
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
                   as_tensor: bool = False) -> FunmResult:
    """d ~ diag f(A) by Eq. 20:
    d_i = zeta_0 + zeta_1 a_ii + sum_c a_ic <Q_c, C_i>,
    Q_c[j] = sum over visits of j by walks from c of zeta_{k+2} W_k (W_0 = 1/N_c)."""
    cfg = check_config(config)
    coeffs = as_stream(coeffs)
    n, nnz = _n_nnz(a)
    z = coeffs.prefix(cfg.max_steps + 2)
    mode = "replay" if replay is not None else "philox"
    if nnz == 0:  # A = 0 -> d = zeta_0 exactly
        return FunmResult(np.full(n, z[0]), "diag", config=_cfg_echo(cfg, coeffs, mode))
    g = _graph(a, device)
    params = WalkParams(cfg, z, g.device)
    ni, pre = _budgets(g, cfg, replay, budgets)
    pcol = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
    st = g.new_stats()
    if replay is None:
        g.walk_diag(params, pre, pcol, stats=st)
    else:
        off, ent = _replay_tensors(g, replay)
        g.replay_diag(params, pre, off, ent, pcol, stats=st)
    d = g.diag_combine(z[0], z[1], pcol)
    res = FunmResult(d if as_tensor else d.cpu().numpy(), "diag", config=_cfg_echo(cfg, coeffs, mode))
    _stats(res, st)
    res.aux = {"pcol": pcol, "ni": ni, "walk_pre": pre}
    return res
