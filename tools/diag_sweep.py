"""Diag combine tuning sweep (one process, one graph): time one estimate per
environment setting and check every setting gives bit-identical d.

    python tools/diag_sweep.py --config 3 'MCF_DIAG_CHUNK_Q=256,MCF_DIAG_LONG_WORK_Q=256' ...
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("settings", nargs="*")
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2308_01037_b200 as mc
    from paper_2308_01037_b200.device import DeviceGraph, WalkParams

    cfg = dict(bench.CONFIGS[args.config])
    a, beta, n_walks = bench.make_graph(cfg, pinned=True)
    g = DeviceGraph(a, gamma=beta)
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    z = mc.EXPONENTIAL.prefix(cfg["max_steps"] + 2)
    params = WalkParams(wcfg, z)
    from paper_2308_01037_b200 import _native
    params.c.flags = _native.MCF_FLAG_TIME_KERNELS
    ni, pre = g.allocate(n_walks)
    base_env = {k: os.environ.get(k) for k in os.environ if k.startswith("MCF_")}
    ref = None
    for s in [""] + args.settings:
        env = dict(kv.split("=") for kv in s.split(",") if kv)
        for k in list(os.environ):
            if k.startswith("MCF_") and k not in base_env:
                del os.environ[k]
        os.environ.update(env)
        times = []
        for r in range(args.reps + 1):
            pcol = torch.zeros(g.nnz, dtype=torch.float64, device=g.device)
            st = g.new_stats()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.walk_diag(params, pre, pcol, stats=st)
            e1.record()
            torch.cuda.synchronize()
            wk, qk, nl = g.kernel_times(reset=True)
            if r:
                times.append((e0.elapsed_time(e1), wk, qk))
        d = g.diag_combine(z[0], z[1], pcol)
        same = None
        if ref is None:
            ref = d.clone()
        else:
            same = bool(torch.equal(ref, d))
        best = min(times) if times else (0.0, 0.0, 0.0)
        print(json.dumps({"setting": s or "default", "ms": best[0], "walk_ms": best[1], "combine_ms": best[2],
                          "bitwise_same": same}), flush=True)


if __name__ == "__main__":
    main()
