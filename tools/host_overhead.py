"""Host-side cost of one eager estimator call (config 2, resident graph):
wall time per call with a sync, and a cProfile of the Python layer."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2308_01037_b200 as mc  # noqa: E402
from paper_2308_01037_b200 import parallel  # noqa: E402
from paper_2308_01037_b200.device import DeviceGraph  # noqa: E402


def main():
    cfg = bench.CONFIGS[2]
    a, beta, n_walks = bench.make_graph(cfg)
    g = DeviceGraph(a, gamma=beta)
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    for _ in range(5):
        parallel.sharded_action(g, mc.EXPONENTIAL, None, wcfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        parallel.sharded_action(g, mc.EXPONENTIAL, None, wcfg)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ts.append((t1 - t0, t2 - t0))
    ts.sort(key=lambda x: x[1])
    mid = ts[len(ts) // 2]
    print(f"eager call: host enqueue {mid[0] * 1e6:.0f} us, enqueue+complete {mid[1] * 1e6:.0f} us")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(30):
        parallel.sharded_action(g, mc.EXPONENTIAL, None, wcfg)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__":
    main()
