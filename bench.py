#!/usr/bin/env python
"""Benchmark of the walk-sampling estimator (BASELINE.json metric: walk-steps/s
and nodes/s; achieved HBM GB/s vs peak).

Default workload = BASELINE configs[1] ("config 2"): total communicability
exp(beta A) 1 on a Barabasi-Albert graph, n = 1e6, m = 4, beta = 1/lambda_max,
30 Taylor terms (max_steps = 28), 10,000 batches x 64 = 640,000 walks.
A "step" is one full estimator pass: walk budgets, r = A v (v = 1: the row
sums), the walks, the per-column reduction and y = z0 v + z1 r + A q.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|1] [--impl mcfunm|reference]

Under torchrun (N > 1) the start columns are sharded over the ranks and the
per-column results assembled with NCCL (paper_2308_01037_b200/parallel.py).
Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
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
    2: dict(workload="config2: total communicability exp(beta A) 1, Barabasi-Albert n=1e6 m=4, "
                     "beta=1/lambda_max, 30 Taylor terms, 10,000 batches x 64 walks",
            kind="action", graph="ba", n=1_000_000, m=4, n_walks=640_000, max_steps=28, cutoff=1e-300, seed=0),
    1: dict(workload="config1: subgraph centrality diag(exp(beta A)), Erdos-Renyi n=1e4 mean degree 8 (LCC), "
                     "beta=1/lambda_max, 30 Taylor terms, 1000 walks per node",
            kind="diag", graph="er", n=10_000, deg=8, walks_per_node=1000, max_steps=28, cutoff=1e-300, seed=0),
    3: dict(workload="config3: subgraph centrality diag(exp(beta A)), symmetrised R-MAT scale 22 edge factor 16 "
                     "(.57,.19,.19,.05), no loops/duplicates, beta=1/lambda_max, 25 Taylor terms, 200 walks per node",
            kind="diag", graph="rmat", scale=22, ef=16, walks_per_node=200, max_steps=23, cutoff=1e-300, seed=0),
    5: dict(workload="config5: subgraph centrality diag(exp(beta A)), Chung-Lu n=1.6e7 exponent 2.1 mean degree 20 "
                     "max degree 1e5, beta=1/lambda_max, 25 Taylor terms, 100 walks per node",
            kind="diag", graph="chunglu", n=16_000_000, walks_per_node=100, max_steps=23, cutoff=1e-300, seed=0),
    4: dict(workload="config4: Katz resolvent (I - gamma A)^-1 1, symmetrised R-MAT scale 24 edge factor 16 "
                     "(.57,.19,.19,.05), no loops/duplicates, gamma=0.85/lambda_max, W_c=1e-8, 100 walks per node",
            kind="action", graph="rmat", scale=24, ef=16, walks_per_node=100, max_steps=10_000, cutoff=1e-8, seed=0,
            func="resolvent", gamma_frac=0.85),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def make_graph(cfg, pinned=False, scale=None):
    """Host SparseMatrix (for the e2e leg), the scale factor (beta, or the Katz
    gamma) and N_s.  R-MAT configs are generated on the GPU and copied to
    pinned host memory once (setup, untimed)."""
    from paper_2308_01037_b200 import graphs
    if cfg["graph"] in ("rmat", "chunglu"):
        import torch
        from paper_2308_01037_b200.device import DeviceGraph
        from paper_2308_01037_b200.sparsemat import SparseMatrix
        sc = scale or cfg.get("scale")
        if cfg["graph"] == "rmat":
            n, rp, ci = graphs.rmat_device(sc, cfg["ef"], seed=cfg["seed"])
        else:
            n, rp, ci = graphs.chung_lu_device(cfg["n"], seed=cfg["seed"])
        g1 = DeviceGraph.from_device_arrays(n, rp, ci, torch.ones(ci.numel(), dtype=torch.float64, device=rp.device))
        lam = graphs.lambda_max_device(g1)
        g1.close()
        host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (rp, ci)]
        host[0].copy_(rp)
        host[1].copy_(ci)
        vals = torch.ones(ci.numel(), dtype=torch.float64, pin_memory=True)
        a = SparseMatrix.from_csr_arrays(n, host[0].numpy(), host[1].numpy(), vals.numpy(), symmetric_hint=True,
                                         meta={"generator": cfg["graph"], "scale": sc, "lambda_max": lam})
        a._pinned = (host, vals)
        del rp, ci
        torch.cuda.empty_cache()
        scale_factor = cfg.get("gamma_frac", 1.0) / lam
    elif cfg["graph"] == "ba":
        a = graphs.barabasi_albert(cfg["n"], cfg["m"], seed=cfg["seed"], pinned=pinned)
        scale_factor = 1.0 / graphs.lambda_max(a)
    else:
        a = graphs.erdos_renyi_lcc(cfg["n"], cfg["deg"], seed=cfg["seed"])
        scale_factor = 1.0 / graphs.lambda_max(a)
    n_walks = cfg.get("n_walks") or cfg["walks_per_node"] * a.n
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
# CPU legs (oracle port of the reference, sampled)
# --------------------------------------------------------------------------
_CPU = {}


def _cpu_worker(cols):
    from oracle import port
    g = _CPU
    t0 = time.perf_counter()
    if g["kind"] == "action":
        _, em = port.action_columns(g["t"], g["r"], g["z"], g["ni"], cols, g["max_steps"], g["cutoff"], g["seed"])
    else:
        _, em = port.diag_columns(g["A"], g["t"], g["z"], g["ni"], cols, g["max_steps"], g["cutoff"], g["seed"])
    return em, time.perf_counter() - t0


class CpuBaseline:
    """The reference's CPU algorithm (oracle/port.py restatement, same
    PCG64DXSM streams and searchsorted walker) over a bounded, evenly spaced
    sample of the walked columns, on all host cores (fork pool)."""

    def __init__(self, a, beta, n_walks, cfg, cores=None):
        import multiprocessing as mp
        from oracle import port
        t0 = time.perf_counter()
        A = port.Csr.from_any(a).scaled(beta)
        t = port.transition_tables(A)
        ni = port.allocate(t, n_walks)
        z = port.zeta_prefix(cfg.get("func", "exponential"), cfg["max_steps"] + 2)
        _CPU.update(kind=cfg["kind"], t=t, A=A, ni=ni, z=z, r=A.scipy_csr() @ np.ones(A.n),
                    max_steps=cfg["max_steps"], cutoff=cfg["cutoff"], seed=cfg["seed"])
        self.setup_s = time.perf_counter() - t0
        self.walked = np.flatnonzero(ni)
        self.ni = ni
        self.n = A.n
        self.total_emissions_est = None
        self.cores = cores or os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.cores)
        # calibrate: per-column cost on a small evenly spaced probe
        probe = self.walked[:: max(1, self.walked.size // 256)][:256]
        em, dt = _cpu_worker(probe)
        self.sec_per_col = dt / max(1, probe.size)
        self.em_per_col = em / max(1, probe.size)

    def run(self, budget_s):
        k = int(min(self.walked.size, max(self.cores, self.cores * budget_s / max(self.sec_per_col, 1e-9))))
        cols = self.walked[np.linspace(0, self.walked.size - 1, k).astype(np.int64)]
        chunks = np.array_split(cols, self.cores * 4)
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_worker, chunks)
        wall = time.perf_counter() - t0
        em = sum(r[0] for r in res)
        return em, wall, k

    def describe(self, k):
        return (f"{k} of {self.walked.size} walked start columns (evenly spaced by index), full walks of each "
                f"column, reference PCG64DXSM streams; {self.cores} processes")

    def close(self):
        self.pool.terminate()


# --------------------------------------------------------------------------
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    a, beta, n_walks = make_graph(cfg)
    if cfg["graph"] in ("rmat", "chunglu"):
        print(json.dumps({"impl": "reference", "unavailable": "the reference CPU algorithm needs ~80 GB of host RAM "
                                                              "for this R-MAT graph's numpy tables"}), flush=True)
        return 0
    cpu = CpuBaseline(a, beta, n_walks, cfg)
    per_step = max(2.0, min(15.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu.run(per_step / 4)
    em_tot, wall_tot, k = 0, 0.0, 0
    for _ in range(args.steps):
        em, wall, k = cpu.run(per_step)
        em_tot += em
        wall_tot += wall
    cpu.close()
    value = em_tot / wall_tot
    total_em = cpu.em_per_col * cpu.walked.size
    line = {
        "impl": "reference", "metric": "walk-steps/s", "baseline_metric": BASELINE_METRIC, "value": value,
        "unit": "steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall_tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "nodes_per_s": cpu.n / (total_em / value),
        "config": {"workload": cfg["workload"], "n": int(a.n), "nnz": int(a.nnz), "n_walks": int(n_walks),
                   "beta": beta, "max_steps": cfg["max_steps"], "weight_cutoff": cfg["cutoff"]},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cpu.cores, "kind": "port",
                         "sample": cpu.describe(k)},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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

    t0 = time.perf_counter()
    a, beta, n_walks = make_graph(cfg, pinned=True, scale=args.scale)
    per_gpu_walks = n_walks
    if world > 1 and args.scaling == "weak":
        # weak scaling (the path partitions by start column, run instructions 5):
        # every GPU keeps the config's walk budget, the N-GPU job walks N times
        # as many over the same graph (its estimate has N times the samples)
        n_walks = per_gpu_walks * world
    coeffs = coeff_stream(cfg)
    log(f"[bench] graph n={a.n} nnz={a.nnz} beta={beta:.6e} walks={n_walks} ({time.perf_counter() - t0:.1f}s)")
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    z = coeffs.prefix(cfg["max_steps"] + 2)
    params = WalkParams(wcfg, z)
    g = DeviceGraph(a, gamma=beta)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=g.device)  # > 126 MB L2
    # The write leaves L2 full of DIRTY lines whose write-back would otherwise
    # land inside the next timed step; reading a second buffer of the same size
    # (untimed) evicts them, so each step starts with no input cached and a
    # clean L2 ("write": the write alone).
    sweep = torch.zeros(32 << 20, dtype=torch.int64, device=g.device) if args.flush == "write+read" else None
    sweep_out = torch.empty((), dtype=torch.int64, device=g.device)

    def flush_l2():
        flush.zero_()
        if sweep is not None:
            torch.sum(sweep, dim=0, out=sweep_out)

    # N > 1: the exchange runs in peer memory (mcf_spmv_peer / mcf_diag_combine_peer
    # over CUDA IPC / NVLink) unless --transport nccl; the buffers are mapped once
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

    # One estimator pass has no host synchronisation on the action path, so on
    # one GPU it is captured once as a CUDA graph and replayed per step.
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
    # emissions of the whole job (all ranks) over the timed steps
    em_t = torch.stack([s_[1] for s_ in stats]).sum().to(torch.float64).reshape(1)
    if world > 1:
        dist.all_reduce(em_t)
        t_ms = torch.tensor([ms], dtype=torch.float64, device=g.device)
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        ms = float(t_ms.item())
    em_per_step = float(em_t.item()) / args.steps
    value = em_per_step * args.steps / (ms / 1e3)
    nodes_per_s = g.n * args.steps / (ms / 1e3)

    # ---- dominant kernel roofline -------------------------------------------------------
    peak, peak_src = measured_peak()
    walk_avg_ms = walk_ms_tot / max(1, walk_launches)
    # this rank's launches process its share of a step; diag runs batch a step
    # into several walk launches (emission-buffer budget), each one a slice
    walk_launches_per_step = max(1.0, walk_launches / max(1, args.steps))
    em_per_walk_launch = em_per_step / world / walk_launches_per_step
    achieved = BYTES_PER_STEP * em_per_walk_launch / (walk_avg_ms / 1e3) / 1e9 if walk_avg_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_config{args.config}.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": "k_walk_action" if cfg["kind"] == "action" else "k_walk_emit",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src, "bytes_per_step": BYTES_PER_STEP,
                "kernel_ms_avg": walk_avg_ms, "kernel_share_of_step": (walk_ms_tot / ms) if ms else None,
                "random_sector_ceiling_gsteps": 37.8,
                "note": "algorithmic bytes = 64 B x emissions (row header + sampled entry, SURVEY 8d), kept for "
                        "comparability; on uniform-value graphs the lean layout serves a step with ONE random 8-B "
                        "entry. Random HBM reads top out at ~37.8 G/s on this B200 and each costs a 128-B line "
                        "fill (tools/gups, profiles/r01/gups.txt): HBM-resident graphs (config 4) are bound by "
                        "those fills (~88% of the copy peak in DRAM traffic); L2-resident ones (config 2) by the "
                        "latency of the one dependent load, hence frac > 1 against HBM"}
    roofline["walk_launches_per_step"] = walk_launches_per_step
    # the walk's own ceilings (tools/gups.cu, profiles/r01/gups.txt): one dependent
    # random load per step, 279 G/s when the table is L2-resident, 37.8 G/s from HBM
    if walk_avg_ms > 0:
        ksteps = em_per_walk_launch / (walk_avg_ms / 1e3)
        roofline["kernel_steps_per_s"] = ksteps
        roofline["l2_random_load_ceiling_gsteps"] = 279.2
        roofline["frac_of_l2_random_load_ceiling"] = ksteps / 279.2e9
    if cfg["kind"] == "diag":
        roofline["q_kernel_ms"] = q_ms_tot / max(1, args.steps)
        roofline["combine"] = {
            "kernels": "k_diag_q, k_diag_qc<K>, k_diag_big (Q_c build + Eq. 20 combine)",
            "ms_per_step": q_ms_tot / max(1, args.steps),
            "share_of_step": (q_ms_tot / ms) if ms else None,
            "bound": "probe round trips to shared / distributed shared / L2 tables (DESIGN 6), not DRAM bandwidth"}
    elif q_ms_tot:  # action: the span before the walks (budgets, r) recorded by mcf_funm_action
        roofline["prewalk_ms_avg"] = q_ms_tot / max(1, args.steps)

    # ---- end to end through the public API (host matrix -> host result) --------------
    e2e = None
    if not args.no_e2e:
        h2d = int(a.csr.indptr.nbytes + a.csr.indices.nbytes + a.csr.data.nbytes)
        d2h = 8 * a.n
        e2e_ms = []
        e2e_warm = max(1, args.warmup)  # first calls warm the pinned/device allocators
        for i in range(max(1, args.steps) + e2e_warm):
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
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / len(e2e_ms),
               "nodes_per_s": g.n * len(e2e_ms) / (e_ms / 1e3),
               "path": "DeviceGraph(host SparseMatrix, gamma) + estimator + y to host: pinned H2D of CSR, pinned D2H of y"}

    # ---- CPU baseline (rank 0, N = 1 only) ---------------------------------------------
    cpu = None
    if cfg["graph"] in ("rmat", "chunglu"):
        cpu = {"value": None, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
               "sample": "not run: the oracle's numpy tables for this graph need tens of GB of host RAM (SURVEY §8c)"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        cb = CpuBaseline(a, beta, n_walks, cfg)
        em, wall, k = cb.run(args.cpu_seconds)
        cpu = {"value": em / wall, "unit": "steps/s", "cores": cb.cores, "kind": "port", "sample": cb.describe(k)}
        cb.close()

    if rank == 0:
        line = {
            "metric": "walk-steps/s", "baseline_metric": BASELINE_METRIC, "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "nodes_per_s": nodes_per_s,
            "config": {"workload": cfg["workload"], "n": g.n, "nnz": g.nnz, "n_walks": int(n_walks),
                       "walks_per_gpu": int(n_walks // world),
                       "emissions_per_step": em_per_step, "beta": beta, "max_steps": cfg["max_steps"],
                       "weight_cutoff": cfg["cutoff"], "seed": cfg["seed"], "sampling": "philox (device RNG)",
                       "l2": ("flushed between timed steps (untimed): 256 MiB write, then a 256 MiB read of another "
                              "buffer to evict the dirty lines" if args.flush == "write+read" else
                              "flushed between timed steps (256 MiB write, untimed)"),
                       "parallelism": f"start-column shards x{world}, graph replicated"
                                      + (f", exchange: {args.transport}" if world > 1 else "")},
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mcfunm", choices=["mcfunm", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--flush", choices=["write", "write+read"], default="write")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N > 1 exchange: peer-memory combine kernels (default) or NCCL all-reduce")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager steps instead of a captured CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--scale", type=int, default=None, help="override the R-MAT scale (config 4)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N > 1: weak = every GPU keeps the config's walk budget (default); strong = the config's "
                         "budget split over the GPUs")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.scale and cfg["graph"] == "rmat":
        cfg["scale"] = args.scale
        cfg["workload"] = cfg["workload"].replace("scale 24", f"scale {args.scale}")
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_device(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
