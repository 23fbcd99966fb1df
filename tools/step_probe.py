"""Critical-path probe for the config-2 action step: CUDA-graph replay time of
the full mcf_funm_action and of its pieces (cold L2 before every replay)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2308_01037_b200 as mc  # noqa: E402
from paper_2308_01037_b200.device import DeviceGraph, WalkParams  # noqa: E402


def timed(fn, flush, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    cfg = bench.CONFIGS[2]
    a, beta, n_walks = bench.make_graph(cfg)
    g = DeviceGraph(a, gamma=beta)
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    z = mc.EXPONENTIAL.prefix(cfg["max_steps"] + 2)
    p = WalkParams(wcfg, z)
    v = torch.ones(g.n, dtype=torch.float64, device=g.device)
    r, q, y = (torch.zeros(g.n, dtype=torch.float64, device=g.device) for _ in range(3))
    ni, pre = g.allocate(n_walks)
    st = g.new_stats()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=g.device)
    res = {
        "funm_action (all)": lambda: g.funm_action(p, n_walks, v, z[0], z[1], r, q, y, stats=st),
        "allocate": lambda: g.allocate(n_walks),
        "spmv r": lambda: g.spmv(v, out=r),
        "walk_action (budgets given)": lambda: g.walk_action(p, pre, r, q, stats=st),
        "spmv combine": lambda: g.spmv(q, alpha=z[0], v=v, beta=z[1], r=r, out=y),
        "spmv+walk+spmv": lambda: (g.spmv(v, out=r), g.walk_action(p, pre, r, q, stats=st),
                                   g.spmv(q, alpha=z[0], v=v, beta=z[1], r=r, out=y)),
        "flush only": lambda: None,
    }
    for k, fn in res.items():
        if k == "flush only":
            continue
        print(f"{k:32s} {timed(fn, flush):8.1f} us", flush=True)


if __name__ == "__main__":
    main()
