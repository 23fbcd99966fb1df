"""Centrality layer of the drop-in.

subgraph_centrality(a, gamma, config)   -> diag(exp(gamma A))
total_communicability(a, gamma, config) -> exp(gamma A) 1
katz_centrality(a, fraction, config)    -> (I - gamma A)^-1 1
The scaling by gamma happens on the device (DeviceGraph(a, gamma)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .device import DeviceGraph
from .errors import ArgumentError, ConvergenceError
from .estimators import FunmResult, rand_funm_action, rand_funm_diag
from .series import EXPONENTIAL, RESOLVENT
from .walker import alpha_diagnostic


@dataclass
class CentralityReport:
    """Scores in original node ids; ranking = ids by descending score, ties by
    ascending id."""

    measure: str
    scores: np.ndarray
    node_ids: np.ndarray
    ranking: np.ndarray
    gamma: float
    stats: dict = field(default_factory=dict)
    result: FunmResult | None = None


def _report(measure, a, scores, gamma, res: FunmResult | None) -> CentralityReport:
    ids = getattr(a, "original_ids", None)
    ids = np.arange(scores.size) if ids is None else np.asarray(ids)
    order = np.lexsort((ids, -scores))
    stats = {}
    if res is not None:
        stats = {"walks": res.walks, "emissions": res.emissions, "mean_steps": res.mean_steps,
                 "truncated": res.truncated, "absorbed": res.absorbed, **res.config}
    return CentralityReport(measure, scores, ids, ids[order], float(gamma), stats, res)


def _check_graph(a):
    n = a.n if isinstance(a, DeviceGraph) else a.csr.shape[0]
    nnz = a.nnz if isinstance(a, DeviceGraph) else a.csr.nnz
    if nnz == 0:
        raise ArgumentError("empty graph: centrality is undefined")
    if isinstance(a, DeviceGraph):
        if not a.symmetric_hint:
            raise ArgumentError("adjacency must be symmetric (symmetrize directed graphs first, Eq. 25)")
    elif not getattr(a, "symmetric_hint", False):
        diff = a.csr - a.csr.T
        if diff.nnz and np.abs(diff.data).max() != 0.0:
            raise ArgumentError("adjacency must be symmetric (symmetrize directed graphs first, Eq. 25)")
    return n


def _scaled(a, gamma, device):
    if not gamma > 0:
        raise ArgumentError(f"gamma must be positive, got {gamma}")
    return a.scaled(gamma) if isinstance(a, DeviceGraph) else DeviceGraph(a, gamma=gamma, device=device)


def subgraph_centrality(a, gamma: float, config, *, device=None, **kw) -> CentralityReport:
    """fSC(i) = exp(gamma A)_ii via rand_funm_diag on scale(a, gamma)."""
    _check_graph(a)
    g = _scaled(a, gamma, device)
    res = rand_funm_diag(g, EXPONENTIAL, config, **kw)
    return _report("subgraph", a, np.asarray(res.values if not torch.is_tensor(res.values) else res.values.cpu()),
                   gamma, res)


def total_communicability(a, gamma: float, config, *, device=None, **kw) -> CentralityReport:
    """fTC(i) = (exp(gamma A) 1)_i via rand_funm_action with v = 1."""
    n = _check_graph(a)
    g = _scaled(a, gamma, device)
    res = rand_funm_action(g, EXPONENTIAL, None, config, **kw)  # v = 1
    return _report("total-communicability", a,
                   np.asarray(res.values if not torch.is_tensor(res.values) else res.values.cpu()), gamma, res)


def gershgorin_gamma(a, fraction: float) -> float:
    """fraction / max row |a| sum (reference oracle.py:128-136)."""
    if not (0.0 < fraction < 1.0):
        raise ArgumentError("fraction must lie strictly between 0 and 1")
    if isinstance(a, DeviceGraph):
        m = a.info["max_row_abs_sum"]
    else:
        if a.csr.nnz == 0:
            raise ArgumentError("zero matrix has no meaningful attenuation factor")
        rows = np.repeat(np.arange(a.csr.shape[0]), np.diff(a.csr.indptr))
        s = np.zeros(a.csr.shape[0])
        np.add.at(s, rows, np.abs(a.csr.data))
        m = float(s.max())
    return fraction / m


def cg_katz(g: DeviceGraph, b: torch.Tensor, tol: float = 1e-10, max_iter: int = 1000):
    """Unpreconditioned CG on (I - gamma A) x = b, ``g`` holding gamma * A, with
    the device SpMV (reference oracle.py:83-125 semantics; Katz cross-check)."""
    x = torch.zeros_like(b)
    r = b.clone()
    p = r.clone()
    rs = float(r @ r)
    lim = tol * float(torch.linalg.norm(b))
    if math.sqrt(rs) <= lim:
        return x
    ap = torch.empty_like(b)
    for _ in range(max_iter):
        g.spmv(-p, alpha=1.0, v=p, out=ap)  # ap = p - (gamma A) p
        al = rs / float(p @ ap)
        x += al * p
        r -= al * ap
        rn = float(r @ r)
        if math.sqrt(rn) <= lim:
            return x
        p = r + (rn / rs) * p
        rs = rn
    raise ConvergenceError(f"conjugate gradient did not reach tol={tol} in {max_iter} iterations",
                           residual=math.sqrt(rs))


def katz_centrality(a, fraction: float, config, method: str = "randomized", *, gamma: float | None = None,
                    allow_alpha_ge_1: bool = False, device=None, **kw) -> CentralityReport:
    """KC = (I - gamma A)^-1 1 with gamma = fraction / max row sum (Gershgorin,
    SPEC.md:525-533).  ``gamma`` may be given explicitly.  The randomized
    method rejects alpha = (gamma max_i sum_j |a_ij|)^2 >= 1 (SPEC.md:529,
    Theorem 1: the walk series is not guaranteed to converge) unless
    ``allow_alpha_ge_1`` is set -- BASELINE config 4 (gamma = 0.85/lambda_max,
    alpha >> 1) runs that way: its walks still end at the weight cutoff
    (SURVEY.md §3.2), and the estimate is checked against CG."""
    n = _check_graph(a)
    if gamma is None:
        gamma = gershgorin_gamma(a, fraction)
    elif method == "randomized" and not allow_alpha_ge_1:
        m2 = (float(a.info["max_row_abs_sum"]) ** 2 if isinstance(a, DeviceGraph) else alpha_diagnostic(a))
        alpha = float(gamma) ** 2 * m2
        if alpha >= 1.0:
            raise ArgumentError(f"resolvent with alpha = {alpha:.4g} >= 1 after scaling is rejected "
                                "(Theorem 1, SPEC.md:529); pass allow_alpha_ge_1=True to run it anyway")
    g = _scaled(a, gamma, device)
    if method == "randomized":
        res = rand_funm_action(g, RESOLVENT, None, config, **kw)  # v = 1
        vals = res.values.cpu().numpy() if torch.is_tensor(res.values) else res.values
        return _report("katz", a, np.asarray(vals), gamma, res)
    if method == "cg":
        x = cg_katz(g, torch.ones(n, dtype=torch.float64, device=g.device))
        return _report("katz", a, x.cpu().numpy(), gamma, None)
    raise ArgumentError(f"unknown method '{method}'")


def estrada_index(report: CentralityReport) -> float:
    if report.measure != "subgraph":
        raise ArgumentError("Estrada index needs a subgraph-centrality report")
    return float(np.sum(report.scores))


def ranking_correlation(ref: CentralityReport, test: CentralityReport, top_fraction: float) -> float:
    """Pearson correlation of scores over the top ceil(f n) nodes of ``ref``."""
    if not (0.0 < top_fraction <= 1.0):
        raise ArgumentError("top_fraction must lie in (0, 1]")
    k = int(math.ceil(top_fraction * ref.scores.size))
    if k < 2:
        raise ArgumentError("need at least two selected nodes")
    pos = {int(i): j for j, i in enumerate(ref.node_ids)}
    sel = np.array([pos[int(i)] for i in ref.ranking[:k]])
    tpos = {int(i): j for j, i in enumerate(test.node_ids)}
    tsel = np.array([tpos[int(ref.node_ids[j])] for j in sel])
    return float(np.corrcoef(ref.scores[sel], test.scores[tsel])[0, 1])
