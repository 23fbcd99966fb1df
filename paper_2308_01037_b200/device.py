"""Device-resident graph: CSR/CSC arrays in HBM plus the C-ABI handle that owns
the derived transition tables (node headers, packed column ids, row CDFs,
column norms, start distribution).

PyTorch only provides device memory and the stream; every computation is a
kernel of libmcfunm_cuda.so called through ``_native``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import ArgumentError, DegenerateInputError, DeviceError


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the estimator runs only on the GPU (no CPU fallback)")
    N.lib()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ArgumentError(f"device must be a CUDA device, got {dev}")
    return dev


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy through a page-locked buffer (the copy runs at
    PCIe DMA speed instead of staging through pageable memory)."""
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()


def _same_storage(csr, csc) -> bool:
    """CSC arrays of a symmetric matrix that are (or equal) the CSR arrays."""
    if csc.indptr is csr.indptr and csc.indices is csr.indices and csc.data is csr.data:
        return True
    return (csc.indptr.shape == csr.indptr.shape and csc.indices.shape == csr.indices.shape
            and np.array_equal(csc.indptr, csr.indptr) and np.array_equal(csc.indices, csr.indices)
            and np.array_equal(csc.data, csr.data))


def _upload(arr, dtype, dev) -> torch.Tensor:
    """Host array -> device tensor (one H2D copy; page-locked sources DMA directly)."""
    a = np.ascontiguousarray(arr, dtype=dtype)
    return torch.from_numpy(a).to(dev, non_blocking=False)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


_ZETA_CACHE: dict = {}  # (device, coefficient bytes) -> device table; the tables are constants


def _zeta_table(z: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Device copy of a coefficient prefix, made once per (device, values):
    a fresh pageable copy per call would synchronise the host with the stream."""
    key = (str(dev), z.tobytes())
    t = _ZETA_CACHE.get(key)
    if t is None:
        if len(_ZETA_CACHE) > 256:
            _ZETA_CACHE.clear()
        t = torch.from_numpy(z.copy()).to(dev)
        _ZETA_CACHE[key] = t
    return t


class WalkParams:
    """mcf_walk_params for one configuration; holds the device zeta table.

    walk_capacity = N_s bounds the walks of any column range, which lets the
    library size its buffers without reading the budgets back (no host sync:
    a whole estimator pass can be captured in a CUDA graph)."""

    def __init__(self, config, zeta: np.ndarray, device=None):
        z = np.ascontiguousarray(zeta, dtype=np.float64)
        if z.size < config.max_steps + 2:
            raise ArgumentError("zeta table shorter than max_steps + 2")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.zeta = _zeta_table(z, dev)
        self.c = N.McfWalkParams(int(config.max_steps), float(config.weight_cutoff),
                                 int(config.seed) & 0xFFFFFFFFFFFFFFFF, self.zeta.data_ptr(),
                                 int(config.n_walks), 0)

    def derive(self, capacity: int | None = None, flags: int | None = None) -> "WalkParams":
        """A copy with another walk_capacity (the exact walk count of a call:
        a shard's walks, or the sum of explicit budgets; 0 = read it on the
        device) and/or flags; shares the device zeta table."""
        out = WalkParams.__new__(WalkParams)
        out.zeta = self.zeta
        c = self.c
        out.c = N.McfWalkParams(c.max_steps, c.weight_cutoff, c.seed, c.zeta,
                                c.walk_capacity if capacity is None else int(capacity),
                                c.flags if flags is None else int(flags))
        return out


class DeviceGraph:
    """Square sparse matrix on one GPU, scaled by ``gamma`` on the device.

    ``a`` is any object with scipy ``.csr``/``.csc`` arrays (this package's or
    the reference's SparseMatrix).  A matrix with ``symmetric_hint`` whose CSC
    arrays equal its CSR arrays is uploaded once and the CSC view aliases it.
    """

    def __init__(self, a, gamma: float = 1.0, device=None):
        self.device = require_cuda(device)
        csr, csc = a.csr, a.csc
        self.n = int(csr.shape[0])
        self.nnz = int(csr.nnz)
        if self.nnz == 0:
            raise DegenerateInputError("all columns are zero: the initial distribution is undefined")
        if not gamma > 0:
            raise ArgumentError(f"gamma must be positive, got {gamma}")
        self.gamma = float(gamma)
        self.symmetric_hint = bool(getattr(a, "symmetric_hint", False))
        if not csr.has_sorted_indices:
            csr = csr.sorted_indices()
        dev = self.device
        self.row_ptr = _upload(csr.indptr, np.int64, dev)
        self.col_ids = _upload(csr.indices, np.int32, dev)
        self.vals = _upload(csr.data, np.float64, dev)
        same = self.symmetric_hint and _same_storage(csr, csc)
        if same:
            self.csc_ptr, self.csc_rows, self.csc_vals = self.row_ptr, self.col_ids, self.vals
        else:
            if not csc.has_sorted_indices:
                csc = csc.sorted_indices()
            self.csc_ptr = _upload(csc.indptr, np.int64, dev)
            self.csc_rows = _upload(csc.indices, np.int32, dev)
            self.csc_vals = _upload(csc.data, np.float64, dev)
        if self.gamma != 1.0:  # scale() on the device, in place (the uploads are our own copies)
            self.vals.mul_(self.gamma)
            if not same:
                self.csc_vals.mul_(self.gamma)
        self.aliased = same
        self._build()

    @classmethod
    def from_device_arrays(cls, n, row_ptr, col_ids, vals, csc_ptr=None, csc_rows=None, csc_vals=None,
                           symmetric=True):
        """Adopt arrays that already live on the GPU (graph generators, benches)."""
        self = cls.__new__(cls)
        self.device = require_cuda(row_ptr.device)
        self.n = int(n)
        self.nnz = int(col_ids.numel())
        if self.nnz == 0:
            raise DegenerateInputError("all columns are zero: the initial distribution is undefined")
        self.gamma = 1.0
        self.symmetric_hint = bool(symmetric)
        self.row_ptr = row_ptr.to(torch.int64).contiguous()
        self.col_ids = col_ids.to(torch.int32).contiguous()
        self.vals = vals.to(torch.float64).contiguous()
        if csc_ptr is None:
            if not symmetric:
                raise ArgumentError("non-symmetric input needs CSC arrays")
            self.csc_ptr, self.csc_rows, self.csc_vals = self.row_ptr, self.col_ids, self.vals
            self.aliased = True
        else:
            self.csc_ptr = csc_ptr.to(torch.int64).contiguous()
            self.csc_rows = csc_rows.to(torch.int32).contiguous()
            self.csc_vals = csc_vals.to(torch.float64).contiguous()
            self.aliased = False
        self._build()
        return self

    def scaled(self, gamma: float) -> "DeviceGraph":
        """New handle over gamma * A (device multiply, structure shared)."""
        if not gamma > 0:
            raise ArgumentError(f"gamma must be positive, got {gamma}")
        vals = self.vals * gamma
        if self.aliased:
            out = DeviceGraph.from_device_arrays(self.n, self.row_ptr, self.col_ids, vals, symmetric=True)
        else:
            out = DeviceGraph.from_device_arrays(self.n, self.row_ptr, self.col_ids, vals, self.csc_ptr,
                                                 self.csc_rows, self.csc_vals * gamma, self.symmetric_hint)
        out.gamma = self.gamma * gamma
        return out

    # ------------------------------------------------------------------
    def _build(self):
        self._csr = N.McfCsr(self.n, self.nnz, _ptr(self.row_ptr), _ptr(self.col_ids), _ptr(self.vals),
                             _ptr(self.csc_ptr), _ptr(self.csc_rows), _ptr(self.csc_vals))
        h = C.c_void_p()
        N.check(N.lib().mcf_graph_create(C.byref(self._csr), self.stream, C.byref(h)), "mcf_graph_create")
        self.handle = h
        info = N.McfGraphInfo()
        N.check(N.lib().mcf_graph_get_info(h, C.byref(info)), "mcf_graph_get_info")
        self.info = {f: getattr(info, f) for f, _ in info._fields_}

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def close(self):
        h = getattr(self, "handle", None)
        if h:
            N.lib().mcf_graph_destroy(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _f64(self, n=None):
        return torch.empty(self.n if n is None else n, dtype=torch.float64, device=self.device)

    def kernel_times(self, reset: bool = True):
        """(walk-kernel ms, Q-kernel ms, timed walk launches) recorded with
        MCF_FLAG_TIME_KERNELS; reset=False keeps the events (CUDA-graph replays)."""
        w, q, k = C.c_double(), C.c_double(), C.c_int64()
        N.check(N.lib().mcf_graph_kernel_times(self.handle, C.byref(w), C.byref(q), C.byref(k), int(reset)),
                "mcf_graph_kernel_times")
        return w.value, q.value, k.value

    def new_stats(self):
        return torch.zeros(N.MCF_STATS_LEN, dtype=torch.int64, device=self.device)

    # ------------------------------------------------------------------ tables
    def tables(self) -> dict:
        rs, cn, ip = self._f64(), self._f64(), self._f64()
        N.check(N.lib().mcf_graph_tables(self.handle, _ptr(rs), _ptr(cn), _ptr(ip), self.stream), "tables")
        return {"row_abs_sum": rs, "col_norms": cn, "init_prob": ip}

    def diagonal(self) -> torch.Tensor:
        rows = torch.repeat_interleave(torch.arange(self.n, device=self.device), self.row_ptr.diff())
        d = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        on = rows == self.col_ids.to(torch.int64)
        d[rows[on]] = self.vals[on]
        return d

    # ------------------------------------------------------------------ budgets
    def allocate(self, n_walks: int):
        ni = torch.empty(self.n, dtype=torch.int64, device=self.device)
        pre = torch.empty(self.n + 1, dtype=torch.int64, device=self.device)
        N.check(N.lib().mcf_allocate_walks(self.handle, int(n_walks), _ptr(ni), _ptr(pre), self.stream),
                "mcf_allocate_walks")
        return ni, pre

    def budgets(self, ni):
        ni = torch.as_tensor(np.asarray(ni, dtype=np.int64)).to(self.device)
        if ni.numel() != self.n or bool((ni < 0).any()):
            raise ArgumentError("walk budgets must be n non-negative integers")
        pre = torch.zeros(self.n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(ni, 0, out=pre[1:])
        return ni, pre

    # ------------------------------------------------------------------ kernels
    def spmv(self, x, alpha=0.0, v=None, beta=0.0, r=None, out=None, rows=None):
        """y = alpha v + beta r + A x; x None: y = A 1 as CSR-order row sums
        (bit-identical to the reference's A @ ones)."""
        out = self._f64() if out is None else out
        rb, re = (0, self.n) if rows is None else rows
        N.check(N.lib().mcf_spmv(self.handle, float(alpha), _ptr(v), float(beta), _ptr(r), _ptr(x), _ptr(out),
                                 int(rb), int(re), self.stream), "mcf_spmv")
        return out

    def spmv_peer(self, x_parts, bounds, y_outs, alpha=0.0, v=None, beta=0.0, r=None, rows=None):
        """y = alpha v + beta r + A x with x gathered from per-part device
        buffers (x_parts[k] owns indices [bounds[k], bounds[k+1])) and every
        row stored to every buffer in y_outs (raw device pointers, local or
        mapped peer memory; mcf_spmv_peer)."""
        rb, re = (0, self.n) if rows is None else rows
        xs = (C.c_void_p * len(x_parts))(*[int(p) for p in x_parts])
        bs = (C.c_int64 * len(bounds))(*[int(b) for b in bounds])
        ys = (C.c_void_p * len(y_outs))(*[int(p) for p in y_outs])
        N.check(N.lib().mcf_spmv_peer(self.handle, float(alpha), _ptr(v), float(beta), _ptr(r), xs, bs, len(x_parts),
                                      ys, len(y_outs), int(rb), int(re), self.stream), "mcf_spmv_peer")

    def walk_action(self, params: WalkParams, walk_pre, r, q, qvar=None, cols=None, stats=None):
        cb, ce = (0, self.n) if cols is None else cols
        N.check(N.lib().mcf_walk_action(self.handle, C.byref(params.c), _ptr(walk_pre), int(cb), int(ce), _ptr(r),
                                        _ptr(q), _ptr(qvar), _ptr(stats), self.stream), "mcf_walk_action")

    def funm_action(self, params: WalkParams, n_walks: int, v, z0, z1, r, q, y, qvar=None, stats=None,
                    ni=None, walk_pre=None, want_ni: bool = True):
        """Whole single-process RandFunmAction pass in one library call: the
        budgets for n_walks, r = A v (v None: v = 1), walks, q and y.  Returns
        (y, ni, walk_pre); ni is None when want_ni is False (not stored)."""
        if ni is None and want_ni:
            ni = torch.empty(self.n, dtype=torch.int64, device=self.device)
        walk_pre = torch.empty(self.n + 1, dtype=torch.int64, device=self.device) if walk_pre is None else walk_pre
        N.check(N.lib().mcf_funm_action(self.handle, C.byref(params.c), int(n_walks), _ptr(ni), _ptr(walk_pre),
                                        _ptr(v), float(z0), float(z1), _ptr(r), _ptr(q), _ptr(qvar), _ptr(y),
                                        _ptr(stats), self.stream), "mcf_funm_action")
        return y, ni, walk_pre

    def replay_action(self, params: WalkParams, walk_pre, walk_off, entries, r, q, cols=None, stats=None):
        cb, ce = (0, self.n) if cols is None else cols
        N.check(N.lib().mcf_replay_action(self.handle, C.byref(params.c), _ptr(walk_pre), int(cb), int(ce),
                                          _ptr(walk_off), _ptr(entries), _ptr(r), _ptr(q), _ptr(stats),
                                          self.stream), "mcf_replay_action")

    def walk_diag(self, params: WalkParams, walk_pre, pcol, cols=None, stats=None):
        cb, ce = (0, self.n) if cols is None else cols
        N.check(N.lib().mcf_walk_diag(self.handle, C.byref(params.c), _ptr(walk_pre), int(cb), int(ce), _ptr(pcol),
                                      _ptr(stats), self.stream), "mcf_walk_diag")

    def replay_diag(self, params: WalkParams, walk_pre, walk_off, entries, pcol, cols=None, stats=None):
        cb, ce = (0, self.n) if cols is None else cols
        N.check(N.lib().mcf_replay_diag(self.handle, C.byref(params.c), _ptr(walk_pre), int(cb), int(ce),
                                        _ptr(walk_off), _ptr(entries), _ptr(pcol), _ptr(stats), self.stream),
                "mcf_replay_diag")

    def walk_qdense(self, params: WalkParams, walk_pre, Q, cols, stats=None):
        """Dense rows Q[c - cols[0], :] of the walk matrix for c in cols."""
        cb, ce = cols
        N.check(N.lib().mcf_walk_qdense(self.handle, C.byref(params.c), _ptr(walk_pre), int(cb), int(ce), _ptr(Q),
                                        int(Q.stride(0)), _ptr(stats), self.stream), "mcf_walk_qdense")
        return Q

    def funm_full(self, params: WalkParams, walk_pre, z0, z1, F, block: int = 1024, stats=None):
        """F = z0 I + z1 A + A Q A (dense row-major F, n x n) with the sparse A
        products in the library (mcf_funm_full)."""
        N.check(N.lib().mcf_funm_full(self.handle, C.byref(params.c), _ptr(walk_pre), float(z0), float(z1), _ptr(F),
                                      int(F.stride(0)), int(block), _ptr(stats), self.stream), "mcf_funm_full")
        return F

    def diag_combine_peer(self, z0, z1, pcol_parts, col_bounds, d_outs, rows=None):
        """d over a row range with pcol[(i, c)] read from the part owning
        column c and every d_i stored to every buffer in d_outs (raw device
        pointers, local or mapped peer memory; mcf_diag_combine_peer)."""
        rb, re = (0, self.n) if rows is None else rows
        xs = (C.c_void_p * len(pcol_parts))(*[int(p) for p in pcol_parts])
        bs = (C.c_int64 * len(col_bounds))(*[int(b) for b in col_bounds])
        ys = (C.c_void_p * len(d_outs))(*[int(p) for p in d_outs])
        N.check(N.lib().mcf_diag_combine_peer(self.handle, float(z0), float(z1), xs, bs, len(pcol_parts), ys,
                                              len(d_outs), int(rb), int(re), self.stream), "mcf_diag_combine_peer")

    def column_costs(self, walk_pre, max_steps: int, mode: str = "diag") -> torch.Tensor:
        """Per-column work estimate (int64, device) for cost-balanced shards:
        N_c for action; emissions plus Eq. 20 combine probes for diag."""
        cost = torch.empty(self.n, dtype=torch.int64, device=self.device)
        N.check(N.lib().mcf_column_costs(self.handle, _ptr(walk_pre), int(max_steps), 1 if mode == "diag" else 0,
                                         _ptr(cost), self.stream), "mcf_column_costs")
        return cost

    def diag_variance(self, pcol_groups: torch.Tensor, walk_pre, var=None, rows=None):
        """Var(d_i) from G walk-group partial vectors (pcol_groups: G x nnz)."""
        var = self._f64() if var is None else var
        rb, re = (0, self.n) if rows is None else rows
        N.check(N.lib().mcf_diag_variance(self.handle, _ptr(pcol_groups), int(pcol_groups.shape[0]), _ptr(walk_pre),
                                          _ptr(var), int(rb), int(re), self.stream), "mcf_diag_variance")
        return var

    def diag_combine(self, z0, z1, pcol, d=None, rows=None):
        d = self._f64() if d is None else d
        rb, re = (0, self.n) if rows is None else rows
        N.check(N.lib().mcf_diag_combine(self.handle, float(z0), float(z1), _ptr(pcol), _ptr(d), int(rb), int(re),
                                         self.stream), "mcf_diag_combine")
        return d
