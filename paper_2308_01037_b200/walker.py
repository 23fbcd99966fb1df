"""Walk configuration of the drop-in (reference walker.py:44-67, :293-302).

The walk machinery itself (transition tables, budgets, RNG, the synchronised
batch driver) runs on the device -- see include/mcfunm_cuda.h."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ArgumentError

ABSORBING = -1


@dataclass
class WalkConfig:
    """n_walks: global budget N_s; weight_cutoff: W_c in (0, 1), a walk stops
    once |W| <= W_c W0; max_steps: hard cap; seed: RNG key."""

    n_walks: int
    weight_cutoff: float = 1e-6
    max_steps: int = 10_000
    seed: int = 0

    def __post_init__(self):
        self.n_walks = int(self.n_walks)
        if self.n_walks < 1:
            raise ArgumentError("n_walks must be at least 1")
        if not (0.0 < self.weight_cutoff < 1.0):
            raise ArgumentError("weight_cutoff must lie strictly between 0 and 1")
        if self.max_steps < 1:
            raise ArgumentError("max_steps must be at least 1")


def check_config(cfg) -> WalkConfig:
    """Accept this WalkConfig, the reference's, or anything with the same fields."""
    if isinstance(cfg, WalkConfig):
        return cfg
    try:
        return WalkConfig(cfg.n_walks, cfg.weight_cutoff, cfg.max_steps, cfg.seed)
    except AttributeError as exc:
        raise ArgumentError(f"config lacks WalkConfig field: {exc}") from None


def alpha_diagnostic(a) -> float:
    """max_i (sum_j |a_ij|)^2 (Theorem 1; must be < 1 for the resolvent)."""
    if a.csr.nnz == 0:
        return 0.0
    rows = np.repeat(np.arange(a.csr.shape[0]), np.diff(a.csr.indptr))
    s = np.zeros(a.csr.shape[0])
    np.add.at(s, rows, np.abs(a.csr.data))
    return float(s.max() ** 2)


def largest_remainder(probs, total: int) -> np.ndarray:
    """floor(p N) plus one for the largest remainders, ties by ascending index,
    p == 0 never selected (reference walker.py:148-162 contract).  Host-side,
    for small supports (rand_funm_entry); the full allocation runs on the GPU."""
    p = np.asarray(probs, dtype=np.float64)
    want = p * total
    got = np.floor(want).astype(np.int64)
    left = int(total - got.sum())
    if left > 0:
        rem = want - got
        rem[p == 0.0] = -1.0
        got[np.argsort(-rem, kind="stable")[:left]] += 1
    return got
