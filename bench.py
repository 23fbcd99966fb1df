#!/usr/bin/env python
"""Benchmark of the walk-sampling estimator (BASELINE.json metric: walk-steps/s
and nodes/s; achieved HBM GB/s vs peak).

Default workload (N = 1) = BASELINE configs[2] ("config 3"), the largest
configuration that fits one GPU and the one the metric is quoted on for a
single B200: subgraph centrality diag(exp(beta A)) on a symmetrised R-MAT
graph, scale 22, edge factor 16, beta = 1/lambda_max, 25 Taylor terms
(max_steps = 23), 200 walks per node.  A "step" is one full estimator pass:
walk budgets, the walks, the Q_c rows and the Eq. 20 combine, d.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|1|2|4|5] [--impl mcfunm|reference]

Inputs come from tools/bench_graphs.py: a fixed recipe (numpy / scipy / torch
only), cached so both arms read the same CSR and beta bits.

--impl reference times the reference's own CPU algorithm -- the oracle port
of walker.run_walks_batch (same PCG64DXSM streams, global searchsorted) plus
the restated Eq. 20 / Alg. 3 accumulation -- on all host cores, over a
stratified sample of the walked columns, extrapolated to the full estimate
(BASELINE.md §3).  Under torchrun (N > 1) the device arm shards the start
columns over the ranks (cost-balanced, paper_2308_01037_b200/parallel.py) and
assembles the result in peer memory or over NCCL.  Prints one JSON line on
rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE_METRIC = "walk-steps/s and nodes/s at 1/2/4/8 B200; achieved HBM GB/s vs peak"
BYTES_PER_STEP = 64  # two dependent random 32-B sectors per emitted step

CONFIGS = {
    1: dict(workload="config1: subgraph centrality diag(exp(beta A)), Erdos-Renyi n=1e4 mean degree 8 (LCC), "
                     "beta=1/lambda_max, 30 Taylor terms, 1000 walks per node",
            kind="diag", graph="er", n=10_000, deg=8, walks_per_node=1000, max_steps=28, cutoff=1e-300, seed=0),
    2: dict(workload="config2: total communicability exp(beta A) 1, Barabasi-Albert n=1e6 m=4, "
                     "beta=1/lambda_max, 30 Taylor terms, 10,000 batches x 64 walks",
            kind="action", graph="ba", n=1_000_000, m=4, n_walks=640_000, max_steps=28, cutoff=1e-300, seed=0),
    3: dict(workload="config3: subgraph centrality diag(exp(beta A)), symmetrised R-MAT scale 22 edge factor 16 "
                     "(.57,.19,.19,.05), no loops/duplicates, beta=1/lambda_max, 25 Taylor terms, 200 walks per node",
            kind="diag", graph="rmat", scale=22, ef=16, walks_per_node=200, max_steps=23, cutoff=1e-300, seed=0),
    4: dict(workload="config4: Katz resolvent (I - gamma A)^-1 1, symmetrised R-MAT scale 24 edge factor 16 "
                     "(.57,.19,.19,.05), no loops/duplicates, gamma=0.85/lambda_max, W_c=1e-8, 100 walks per node",
            kind="action", graph="rmat", scale=24, ef=16, walks_per_node=100, max_steps=10_000, cutoff=1e-8, seed=0,
            func="resolvent", gamma_frac=0.85),
    5: dict(workload="config5: subgraph centrality diag(exp(beta A)), Chung-Lu n=1.6e7 exponent 2.1 mean degree 20 "
                     "max degree 1e5, beta=1/lambda_max, 25 Taylor terms, 100 walks per node",
            kind="diag", graph="chunglu", n=16_000_000, walks_per_node=100, max_steps=23, cutoff=1e-300, seed=0),
}
# not a BASELINE config: config 2's graph with signed, non-uniform weights (every row
# non-uniform: the alias-table walk), for the weighted-row measurement
CONFIGS[6] = dict(workload="weighted: exp(beta A) 1 on config 2's Barabasi-Albert n=1e6 m=4 with symmetric weights "
                           "|w| ~ U[0.5, 1.5), 10% negative, beta = 1/spectral radius, 30 Taylor terms, 10 walks per node",
                  kind="action", graph="ba_signed", n=1_000_000, m=4, walks_per_node=10, max_steps=28,
                  cutoff=1e-300, seed=0)
DEFAULT_CONFIG = 3


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def graph_spec(cfg):
    keys = ("graph", "n", "m", "deg", "scale", "ef", "seed")
    return {k: cfg[k] for k in keys if k in cfg}


def make_graph(cfg, pinned=False):
    """Host SparseMatrix of the config's graph (values 1), the scale factor
    (beta = 1/lambda_max, or the Katz gamma) and N_s, from the cached recipe."""
    from paper_2308_01037_b200.sparsemat import SparseMatrix
    from tools import bench_graphs
    t0 = time.perf_counter()
    gd = bench_graphs.load(graph_spec(cfg), log=log)
    n, rp, ci = gd["n"], gd["row_ptr"], gd["col_ids"]
    vals = np.asarray(gd["vals"], dtype=np.float64) if "vals" in gd else np.ones(ci.size)
    if pinned:
        import torch
        bufs = [torch.empty(x.shape, dtype={np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
                                             np.dtype(np.float64): torch.float64}[x.dtype], pin_memory=True)
                for x in (rp, ci, vals)]
        for bt, x in zip(bufs, (rp, ci, vals)):
            bt.numpy()[:] = x
        rp, ci, vals = (bt.numpy() for bt in bufs)
    a = SparseMatrix.from_csr_arrays(n, rp, ci, vals, symmetric_hint=True,
                                     meta={"generator": cfg["graph"], "lambda_max": gd["lambda_max"]})
    if pinned:
        a._pinned = bufs
    scale_factor = cfg.get("gamma_frac", 1.0) / gd["lambda_max"]
    n_walks = cfg.get("n_walks") or cfg["walks_per_node"] * n
    log(f"[bench] graph {cfg['graph']} n={n} nnz={ci.size} lambda_max={gd['lambda_max']:.12g} "
        f"({'cached' if gd.get('cached') else 'generated'}, {time.perf_counter() - t0:.1f}s)")
    return a, scale_factor, n_walks


def coeff_stream(cfg):
    import paper_2308_01037_b200 as mc
    return mc.RESOLVENT if cfg.get("func") == "resolvent" else mc.EXPONENTIAL


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cpu():
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "os_cpu_count": os.cpu_count()}


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler (recipe clocks line); keeps timestamped samples so
    the ones inside the timed region can be selected."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index, period_ms=50):
        import threading
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", str(period_ms), "-i", str(index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True, bufsize=1)
        except Exception:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 10:  # wait for the sampler to run
            time.sleep(0.02)

    def _read(self):
        for ln in self.proc.stdout:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                self.samples.append((time.time(), float(f[0]), float(f[1]), f[3:7]))
            except ValueError:
                pass

    def summary(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        inside = [x for x in self.samples if t0 <= x[0] <= t1]
        note = "samples inside the timed region"
        if not inside:  # region shorter than the sampling period: nearest samples around it
            inside = sorted(self.samples, key=lambda x: min(abs(x[0] - t0), abs(x[0] - t1)))[:2]
            note = "timed region shorter than the sampling period; nearest samples"
        reasons = set()
        for x in inside:
            for nm, val in zip(self.NAMES, x[3]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(x[1] for x in inside) if inside else None,
                "sm_max_mhz": max(x[2] for x in inside) if inside else None, "reasons": sorted(reasons),
                "samples": len(inside), "note": note}

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()


# --------------------------------------------------------------------------
# CPU legs: the reference algorithm (oracle/port.py), stratified column sample
# --------------------------------------------------------------------------
_CPU = {}


def _cpu_worker(task):
    """One chunk of sampled start columns of one stratum: (stratum, columns,
    emissions, CPU seconds).  Runs in a forked worker that shares the tables."""
    from oracle import port
    stratum, cols = task
    g = _CPU
    t0 = time.process_time()
    if g["kind"] == "action":
        _, em = port.action_columns(g["t"], g["r"], g["z"], g["ni"], cols, g["max_steps"], g["cutoff"], g["seed"])
    else:
        out = np.zeros(g["A"].n)
        _, em = port.diag_columns(g["A"], g["t"], g["z"], g["ni"], cols, g["max_steps"], g["cutoff"], g["seed"],
                                  out=out)
    return stratum, len(cols), em, time.process_time() - t0


class CpuBaseline:
    """The reference's CPU algorithm on the host cores: the oracle port of
    walker.py (per-column PCG64DXSM streams, global searchsorted walker,
    walker.py:173-290) plus the restated accumulation and combine (Eq. 20 /
    Alg. 3), one forked worker per core over start-column chunks (the result
    does not depend on the split: every column has its own stream).

    Full estimates take minutes to hours on a CPU, so every run times a
    seeded, cost-stratified sample of the walked columns: the walked columns
    are sorted by their work estimate (walk emissions and, for diag, the Eq.
    20 probes -- the combine dominates on hub columns) and cut into STRATA
    groups of equal total work; each run draws columns from every group.  The
    full single-core time is the size-weighted sum of the per-group CPU time
    per column; the all-core time divides it by the cores times the measured
    parallel efficiency of the run."""

    STRATA = 8

    def __init__(self, a, beta, n_walks, cfg, cores=None):
        import multiprocessing as mp
        from oracle import port
        t0 = time.perf_counter()
        n = int(a.n)
        rp = np.asarray(a.csr.indptr, dtype=np.int64)
        ci = np.asarray(a.csr.indices, dtype=np.int64)
        vals = np.asarray(a.csr.data, dtype=np.float64) * beta
        # symmetric 0/1 graphs: the CSC arrays are the CSR arrays
        A = port.Csr(n, rp, ci, vals, rp, ci, vals)
        t = port.transition_tables(A)
        ni = port.allocate(t, n_walks)
        z = port.zeta_prefix(cfg.get("func", "exponential"), cfg["max_steps"] + 2)
        r = A.scipy_csr() @ np.ones(n) if cfg["kind"] == "action" else None
        _CPU.update(kind=cfg["kind"], t=t, A=A, ni=ni, z=z, r=r, max_steps=cfg["max_steps"], cutoff=cfg["cutoff"],
                    seed=cfg["seed"])
        self.n = n
        self.kind = cfg["kind"]
        self.walked = np.flatnonzero(ni)
        deg = np.diff(rp)
        steps = min(cfg["max_steps"], 64) + 1
        m = ni[self.walked] * steps
        if cfg["kind"] == "diag":  # sum_{i in C_c} min(deg i, m_c) (CSC = CSR: symmetric)
            col_of = np.repeat(np.arange(n), deg)
            probes = np.bincount(col_of, weights=np.minimum(deg[ci], (ni * steps)[col_of]), minlength=n)
            del col_of
            cost = 3 * m + probes[self.walked]
        else:
            cost = m
        order = np.argsort(cost, kind="stable")
        cum = np.cumsum(cost[order].astype(np.float64))
        cuts = np.searchsorted(cum, cum[-1] * np.arange(1, self.STRATA) / self.STRATA)
        self.strata = [g for g in np.split(self.walked[order], cuts) if g.size]
        self.stratum_cost = [float(np.sum(c)) for c in np.split(cost[order], cuts) if c.size]
        self.cores = cores or os.cpu_count() or 1
        self.setup_s = time.perf_counter() - t0
        self.pool = mp.get_context("fork").Pool(self.cores)
        # calibration: CPU seconds per column of every stratum, from one or two
        # columns each (one task per column); refined after every run
        rng = np.random.default_rng(12345)
        probe = [(k, np.array([c])) for k, s in enumerate(self.strata)
                 for c in rng.choice(s, size=min(s.size, 2), replace=False)]
        res = self.pool.map(_cpu_worker, probe, chunksize=1)
        self.obs = np.zeros((len(self.strata), 2))  # per stratum: columns, CPU seconds
        for k, nc, _, c in res:
            self.obs[k] += (nc, c)
        self.runs = []
        self.run_index = 0
        log(f"[cpu] tables {self.setup_s:.1f}s, {self.walked.size} walked columns in {len(self.strata)} strata, "
            f"{self.cores} workers, calibration {self.obs[:, 1].sum():.1f} CPU-s")

    def run(self, budget_s):
        """One timed sample of about ``budget_s`` wall seconds on all cores."""
        rng = np.random.default_rng(1000 + self.run_index)
        self.run_index += 1
        per = budget_s * self.cores / len(self.strata)  # CPU seconds per stratum
        tasks = []
        for k, s in enumerate(self.strata):
            sec_per_col = self.obs[k, 1] / max(1.0, self.obs[k, 0])
            want = int(min(s.size, max(1, round(per / max(sec_per_col, 1e-6)))))
            cols = np.sort(rng.choice(s, size=want, replace=False))
            pieces = max(1, min(want, self.cores))
            tasks += [(k, c) for c in np.array_split(cols, pieces) if c.size]
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, tasks, chunksize=1)
        wall = time.perf_counter() - t0
        for k, nc, _, c in res:
            self.obs[k] += (nc, c)
        self.runs.append((res, wall))
        return res, wall

    def estimate(self, runs=None):
        """Extrapolated full estimate from the recorded sample runs."""
        runs = self.runs if runs is None else runs
        S = len(self.strata)
        cols, em, cpu = np.zeros(S), np.zeros(S), np.zeros(S)
        wall = cpu_all = 0.0
        for res, w in runs:
            wall += w
            for k, nc, e, c in res:
                cols[k] += nc
                em[k] += e
                cpu[k] += c
                cpu_all += c
        size = np.array([s.size for s in self.strata], dtype=np.float64)
        have = cols > 0
        t1 = float(np.sum(size[have] * cpu[have] / cols[have]))
        e_full = float(np.sum(size[have] * em[have] / cols[have]))
        eff = min(1.0, cpu_all / max(1e-9, wall * self.cores))
        t_all = t1 / (self.cores * eff)
        return {"emissions_full": e_full, "t1_full_s": t1, "t_all_full_s": t_all, "parallel_efficiency": eff,
                "steps_per_s": e_full / t_all, "steps_per_s_1core": e_full / t1, "nodes_per_s": self.n / t_all,
                "sample_columns": int(cols.sum()), "sample_emissions": int(em.sum()), "sample_wall_s": wall,
                "sample_steps_per_s": float(em.sum()) / max(1e-9, wall)}

    def describe(self, est):
        return (f"{est['sample_columns']} sampled start columns (with repetition across runs; {self.walked.size} walked in all) ({est['sample_emissions']:.3g} "
                f"emissions, {est['sample_wall_s']:.1f} s wall on {self.cores} processes), seeded and stratified "
                f"into {len(self.strata)} groups of equal estimated work (walk emissions"
                f"{' + Eq. 20 probes' if self.kind == 'diag' else ''}); full estimate extrapolated by group size "
                f"(parallel efficiency {est['parallel_efficiency']:.2f}); reference algorithm = oracle port "
                f"(PCG64DXSM streams, global searchsorted walker)")

    def close(self):
        self.pool.terminate()


def cpu_line(cb, est):
    return {"value": est["steps_per_s"], "unit": "steps/s", "cores": cb.cores, "kind": "port",
            "sample": cb.describe(est), "value_1core": est["steps_per_s_1core"],
            "nodes_per_s": est["nodes_per_s"], "full_estimate_s_all_cores": est["t_all_full_s"],
            "full_estimate_s_1core": est["t1_full_s"], "sample_steps_per_s": est["sample_steps_per_s"],
            "host": host_cpu(), "tables_s": cb.setup_s}


def config_dict(cfg, n, nnz, n_walks, beta, world, transport):
    """The workload definition, identical in both arms' lines (the driver compares them key by key);
    arm-specific facts (RNG, emission count) sit beside it, not inside."""
    return {"workload": cfg["workload"], "n": int(n), "nnz": int(nnz), "n_walks": int(n_walks),
            "walks_per_gpu": int(n_walks // world), "beta": beta, "max_steps": cfg["max_steps"],
            "weight_cutoff": cfg["cutoff"], "seed": cfg["seed"],
            "l2": "device arm: L2 flushed between timed steps (256 MiB write, untimed), and the graphs of configs "
                  "3-5 exceed L2 anyway; CPU arm: a fresh column sample every step",
            "parallelism": f"start-column shards x{world} (cost-balanced), graph replicated"
                           + (f", exchange: {transport}" if world > 1 else "")}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    a, beta, n_walks = make_graph(cfg)
    cpu = CpuBaseline(a, beta, n_walks, cfg)
    per_step = max(4.0, 75.0 / max(1, args.steps))
    for _ in range(args.warmup):
        cpu.run(max(1.0, per_step / 4))
    cpu.runs = []
    for _ in range(args.steps):
        cpu.run(per_step)
    est = cpu.estimate()
    cpu.close()
    value = est["steps_per_s"]
    line = {
        "impl": "reference", "metric": "walk-steps/s", "baseline_metric": BASELINE_METRIC, "value": value,
        "unit": "steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * est["t_all_full_s"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "nodes_per_s": est["nodes_per_s"],
        "config": config_dict(cfg, a.n, a.nnz, n_walks, beta, args.gpus, args.transport),
        "sampling": "PCG64DXSM per-column substreams (the reference's RNG)",
        "cpu_baseline": cpu_line(cpu, est),
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timing": "each step = one stratified sample of the estimate on all host cores; value and ms_per_step are "
                  "the full estimate extrapolated from the K timed samples",
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# device arm
# --------------------------------------------------------------------------
def combine_bytes(g, pre):
    """Algorithmic bytes of the Eq. 20 combine per estimate:
    sum over walked columns c of sum_{a in C_c} (32 + 4 deg a) -- the (i, c)
    entry's CSC offsets and the ids of C_a.  Device reduction (setup only)."""
    import torch
    deg = (g.csc_ptr[1:] - g.csc_ptr[:-1])
    per_col = torch.zeros(g.n, dtype=torch.float64, device=g.device)
    col_of = torch.repeat_interleave(torch.arange(g.n, device=g.device), deg)
    per_col.index_add_(0, col_of, (32 + 4 * deg[g.csc_rows.to(torch.int64)]).to(torch.float64))
    walked = (pre[1:] - pre[:-1]) > 0
    return float(per_col[walked].sum())


def run_device(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2308_01037_b200 as mc
    from paper_2308_01037_b200 import _native, parallel
    from paper_2308_01037_b200.device import DeviceGraph, WalkParams, to_host

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MCF_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo -- a functional
    # check of the N > 1 code path on a one-GPU machine, never a measurement
    shared = os.environ.get("MCF_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _native.lib()

    a, beta, n_walks = make_graph(cfg, pinned=True)
    per_gpu_walks = n_walks
    if world > 1 and args.scaling == "weak":
        # weak scaling: every GPU keeps the config's walk budget, the N-GPU job
        # walks N times as many over the same graph
        n_walks = per_gpu_walks * world
    coeffs = coeff_stream(cfg)
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    z = coeffs.prefix(cfg["max_steps"] + 2)
    params = WalkParams(wcfg, z)
    g = DeviceGraph(a, gamma=beta)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=g.device)  # > 126 MB L2

    def flush_l2():
        flush.zero_()

    peers = None
    if world > 1 and args.transport == "peer":
        peers = parallel.PeerBuffers([8 * g.n if cfg["kind"] == "action" else 8 * g.nnz, 8 * g.n])

    def step():
        if cfg["kind"] == "action":
            if peers is not None:
                return parallel.sharded_action_peer(g, coeffs, None, wcfg, params=params, peers=peers)
            return parallel.sharded_action(g, coeffs, None, wcfg, params=params)  # f(A) 1: v = 1
        if peers is not None:
            return parallel.sharded_diag_peer(g, coeffs, wcfg, params=params, peers=peers)
        return parallel.sharded_diag(g, coeffs, wcfg, params=params)

    clocks = Clocks(local) if rank == 0 else None
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    g.kernel_times(reset=True)

    # One action pass has no host synchronisation, so on one GPU it is captured
    # once as a CUDA graph and replayed per step.
    params.c.flags = _native.MCF_FLAG_TIME_KERNELS
    graph = None
    launches_per_step = None
    if cfg["kind"] == "action" and world == 1 and not args.no_graph:
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            g.kernel_times(reset=True)
            l0 = lib.mcf_kernel_launches()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                static_out = step()
            launches_per_step = lib.mcf_kernel_launches() - l0
            graph.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # fall back to eager steps
            log(f"[bench] CUDA graph capture failed ({exc}); timing eager steps")
            graph = None
            torch.cuda.synchronize()
            g.kernel_times(reset=True)

    # ---- device-resident timed region -------------------------------------------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    walk_ms_tot, q_ms_tot, walk_launches = 0.0, 0.0, 0
    launches0 = lib.mcf_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    for i in range(args.steps):
        flush_l2()
        ev[i][0].record()
        if graph is not None:
            graph.replay()
            st = static_out[1].clone()
        else:
            _, st = step()
        ev[i][1].record()
        stats.append(st)
        if graph is not None:  # read this replay's walk-kernel events
            w_, q_, n_ = g.kernel_times(reset=False)
            walk_ms_tot += w_
            q_ms_tot += q_
            walk_launches += n_
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    launches = (launches_per_step * args.steps if graph is not None
                else lib.mcf_kernel_launches() - launches0)
    clk = clocks.summary(t_wall0, t_wall1) if clocks else None
    if clocks:
        clocks.stop()
    ms = sum(s_.elapsed_time(e_) for s_, e_ in ev)
    w_, q_, n_ = g.kernel_times(reset=True)
    if graph is None:
        walk_ms_tot, q_ms_tot, walk_launches = w_, q_, n_
    params.c.flags = 0
    em_t = torch.stack([s_[1] for s_ in stats]).sum().to(torch.float64).reshape(1)
    if world > 1:
        dist.all_reduce(em_t)
        t_ms = torch.tensor([ms], dtype=torch.float64, device=g.device)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ms = float(t_ms.item())
    em_per_step = float(em_t.item()) / args.steps
    value = em_per_step * args.steps / (ms / 1e3)
    nodes_per_s = g.n * args.steps / (ms / 1e3)

    # ---- rooflines: the walk kernel and (diag) the Eq. 20 combine ------------------------
    # The timed steps overlap batch b + 1's walk (on a few reserved SMs) with batch b's combine, so their
    # kernel intervals overlap and neither kernel has the GPU.  The per-kernel durations the rooflines use come
    # from ONE extra estimate with serial batches (MCF_DIAG_OVERLAP=0), outside the timed region.
    k_steps, k_ms, kernel_timing = args.steps, ms, "the timed steps"
    timed_region_kernels = {"combine_ms_per_step": q_ms_tot / max(1, args.steps),
                            "walk_ms_per_launch": walk_ms_tot / max(1, walk_launches),
                            "walk_launches_per_step": walk_launches / max(1, args.steps),
                            "note": "event-timed inside the timed steps; with the walk / combine overlap the two "
                                    "intervals run side by side on disjoint SMs"}
    if (cfg["kind"] == "diag" and world == 1 and g.n > 24576 and os.environ.get("MCF_DIAG_OVERLAP") is None
            and os.environ.get("MCF_DIAG_UNITS") != "0"):
        os.environ["MCF_DIAG_OVERLAP"] = "0"
        try:
            params.c.flags = _native.MCF_FLAG_TIME_KERNELS
            g.kernel_times(reset=True)
            flush_l2()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            torch.cuda.synchronize()
            walk_ms_tot, q_ms_tot, walk_launches = g.kernel_times(reset=True)
            k_steps, k_ms = 1, e0.elapsed_time(e1)
            kernel_timing = (f"one extra estimate with serial batches ({k_ms:.1f} ms; the timed steps run the next "
                             "batch's walk beside the combine, so their kernel intervals overlap)")
        finally:
            params.c.flags = 0
            del os.environ["MCF_DIAG_OVERLAP"]
    peak, peak_src = measured_peak()
    walk_avg_ms = walk_ms_tot / max(1, walk_launches)
    walk_launches_per_step = max(1.0, walk_launches / max(1, k_steps))
    em_per_walk_launch = em_per_step / world / walk_launches_per_step
    w_ach = BYTES_PER_STEP * em_per_walk_launch / (walk_avg_ms / 1e3) / 1e9 if walk_avg_ms > 0 else None

    def traffic_of(kernel, per="dram_bytes_per_launch"):
        # ncu dram__bytes_read.sum + dram__bytes_write.sum of the same command
        # (tools/gpu_traffic.sh -> profiles/traffic_configN.json)
        tp = os.path.join(ROOT, "profiles", f"traffic_config{args.config}.json")
        if os.path.exists(tp):
            with open(tp) as fh:
                t = json.load(fh)
            return t.get(kernel, {}).get(per) if kernel in t else (
                t.get("dram_bytes_per_launch") if kernel.startswith("k_walk") else None)
        return None

    walk_kernel = "k_walk_action" if cfg["kind"] == "action" else "k_walk_emit"
    # L2-resident walk tables (configs 1, 2: < ~100 MB of CSR ids): the walk runs
    # above "HBM speed" and is bound by dependent L2 loads -- report it against
    # the measured L2 random-load ceiling too (profiles/r01/gups.txt)
    l2_resident = 4 * g.nnz + 16 * g.n < 100 * 2 ** 20
    w_steps = em_per_walk_launch / (walk_avg_ms / 1e3) if walk_avg_ms > 0 else None
    walk = {"bound": "hbm", "kernel": walk_kernel, "achieved": w_ach, "peak": peak, "unit": "GB/s",
            "l2_resident": l2_resident,
            "l2_frac": (w_steps / 279.2e9) if (w_steps and l2_resident) else None,
            # measured DRAM traffic per launch (ncu) over the launch time: what the
            # HBM actually moved -- each random 8-B entry costs a line fill
            "frac": (w_ach / peak) if w_ach else None, "traffic": traffic_of(walk_kernel), "peak_source": peak_src,
            "bytes_per_step": BYTES_PER_STEP, "kernel_ms_avg": walk_avg_ms,
            "launches_per_step": walk_launches_per_step,
            "kernel_share_of_step": (walk_ms_tot / k_ms) if k_ms else None,
            "kernel_steps_per_s": em_per_walk_launch / (walk_avg_ms / 1e3) if walk_avg_ms > 0 else None,
            "l2_random_load_ceiling_gsteps": 279.2, "hbm_random_sector_ceiling_gsteps": 37.8,
            "note": "algorithmic bytes = 64 B x emissions (row header + sampled entry, SURVEY 8d); the lean layout "
                    "serves a step with ONE random 4/8-B entry, so L2-resident graphs run above 'HBM' speed and "
                    "HBM-resident ones are bound by 128-B line fills (profiles/r01/gups.txt)"}
    wt = walk.get("traffic")
    if wt and walk_avg_ms > 0:
        walk["traffic_gbs"] = wt / (walk_avg_ms / 1e3) / 1e9
        walk["traffic_frac"] = walk["traffic_gbs"] / peak
        walk["traffic_bytes_per_step"] = wt / em_per_walk_launch if em_per_walk_launch else None
    roofline = walk
    if cfg["kind"] == "diag":
        _, pre_ = g.allocate(wcfg.n_walks)
        cbytes = combine_bytes(g, pre_)
        c_ms = q_ms_tot / max(1, k_steps)
        c_ach = cbytes / (c_ms / 1e3) / 1e9 if c_ms > 0 else None
        combine = {"bound": "hbm",
                   "kernel": ("k_diag_unit<1024/512/256> (Eq. 20 combine by key-group units)" if g.n > 24576
                              else "k_diag_q (Eq. 20 combine, dense Q_c)"),
                   "achieved": c_ach, "peak": peak, "unit": "GB/s", "frac": (c_ach / peak) if c_ach else None,
                   "traffic": traffic_of("combine", "dram_bytes_per_step"), "traffic_unit": "bytes per step",
                   "peak_source": peak_src,
                   "algorithmic_bytes_per_step": cbytes,
                   "bytes_rule": "sum over walked c of sum_{a in C_c} (32 + 4 deg a) (SURVEY 8d)",
                   "kernel_ms_avg": c_ms, "kernel_share_of_step": (q_ms_tot / k_ms) if k_ms else None,
                   "kernel_timing": kernel_timing, "timed_region_kernels": timed_region_kernels}
        # what actually limits it: the committed ncu capture's pipe utilisation (not measured in this run)
        pp = os.path.join(ROOT, "profiles", "r02", f"ncu_unit_config{args.config}.json")
        if g.n > 24576 and os.path.exists(pp):
            try:
                with open(pp) as f:
                    k = json.load(f)[0]
                pct = lambda key: float(k[key].split()[0])
                combine["limiter"] = {
                    "alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                    "lsu_data_pipe_pct": pct("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
                    "issue_active_pct": pct("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
                    "note": "co-limited by instruction issue and shared-memory wavefronts, not by HBM",
                    "source": "profiles/r02/" + os.path.basename(pp) + " (ncu --set full of one launch)"}
            except (KeyError, ValueError, IndexError, OSError):
                pass
        if c_ms > walk_avg_ms * walk_launches_per_step:  # the dominant phase leads
            roofline = dict(combine)
            roofline["walk"] = walk
        else:
            roofline = dict(walk)
            roofline["combine"] = combine
    elif q_ms_tot:  # action: the span before the walks (budgets, r) recorded by mcf_funm_action
        roofline["prewalk_ms_avg"] = q_ms_tot / max(1, args.steps)

    # ---- end to end through the public API (host matrix -> host result) --------------
    e2e = None
    if not args.no_e2e:
        h2d = int(a.csr.indptr.nbytes + a.csr.indices.nbytes + a.csr.data.nbytes)
        d2h = 8 * a.n
        step_s = ms / args.steps / 1e3
        reps = max(1, args.steps if step_s < 1.0 else min(args.steps, 3))
        e2e_warm = 1 if step_s >= 1.0 else max(1, args.warmup)
        e2e_ms = []
        for i in range(reps + e2e_warm):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            ge = DeviceGraph(a, gamma=beta)
            if cfg["kind"] == "action":
                y, _ = parallel.sharded_action(ge, coeffs, None, wcfg)
            else:
                y, _ = parallel.sharded_diag(ge, coeffs, wcfg)
            host = to_host(y)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t1
            ge.close()
            if i >= e2e_warm:
                e2e_ms.append(dt * 1e3)
            assert np.isfinite(host).all()
        e_ms = sum(e2e_ms)
        if world > 1:
            t_ms = torch.tensor([e_ms], dtype=torch.float64, device=g.device)
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
            e_ms = float(t_ms.item())
        e2e = {"value": em_per_step * len(e2e_ms) / (e_ms / 1e3), "unit": "steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / len(e2e_ms), "reps": len(e2e_ms),
               "nodes_per_s": g.n * len(e2e_ms) / (e_ms / 1e3),
               "path": "DeviceGraph(host SparseMatrix, gamma) + estimator + result to host: pinned H2D of the CSR, "
                       "table build, the estimate, pinned D2H"}

    # ---- CPU baseline (rank 0, N = 1 only) ---------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del g  # the device graph is no longer needed; free host staging before the CPU tables
        torch.cuda.empty_cache()
        cb = CpuBaseline(a, beta, wcfg.n_walks, cfg)
        cb.run(args.cpu_seconds)
        cpu = cpu_line(cb, cb.estimate())
        cb.close()
        n_rows, nnz = a.n, a.nnz
    else:
        n_rows, nnz = g.n, g.nnz

    if rank == 0:
        line = {
            "metric": "walk-steps/s", "baseline_metric": BASELINE_METRIC, "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (tools/bench_graphs.py recipe)",
            "nodes_per_s": nodes_per_s,
            "config": config_dict(cfg, n_rows, nnz, n_walks, beta, world, args.transport),
            "emissions_per_step": em_per_step, "sampling": "philox (device RNG)",
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "timing": "CUDA-graph replay of one full estimator pass" if graph is not None else "eager steps",
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if peers is not None:
        peers.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mcfunm", choices=["mcfunm", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N > 1 exchange: peer-memory combine kernels (default) or NCCL all-gather")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager steps instead of a captured CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=60.0, help="wall seconds of the CPU baseline's sample")
    ap.add_argument("--scale", type=int, default=None, help="override the R-MAT scale (configs 3, 4)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = the config's walk budget split over the GPUs (default: configs 3-5 fix "
                         "walks per node); weak = every GPU keeps the config's budget")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.scale and cfg["graph"] == "rmat":
        cfg["workload"] = cfg["workload"].replace(f"scale {cfg['scale']}", f"scale {args.scale}")
        cfg["scale"] = args.scale
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_device(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
