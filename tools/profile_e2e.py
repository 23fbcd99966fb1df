"""Phase breakdown of one end-to-end call (host SparseMatrix -> host result)
for a bench config; prints wall-clock ms per phase (synchronised)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2308_01037_b200 as mc  # noqa: E402
from paper_2308_01037_b200 import parallel  # noqa: E402
from paper_2308_01037_b200.device import DeviceGraph  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main(config=2, reps=3):
    cfg = bench.CONFIGS[config]
    a, beta, n_walks = bench.make_graph(cfg, pinned=True)
    wcfg = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
    for rep in range(reps):
        ph = {}
        t0 = t()
        rp = torch.from_numpy(a.csr.indptr).to("cuda")
        ci = torch.from_numpy(a.csr.indices).to("cuda")
        va = torch.from_numpy(a.csr.data).to("cuda")
        t1 = t()
        ph["h2d"] = t1 - t0
        g = DeviceGraph.from_device_arrays(a.n, rp, ci, va * beta, symmetric=True)
        t2 = t()
        ph["build"] = t2 - t1
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
        if cfg["kind"] == "action":
            y, st = parallel.sharded_action(g, mc.EXPONENTIAL, None, wcfg)
        else:
            y, st = parallel.sharded_diag(g, mc.EXPONENTIAL, wcfg)
        t3 = t()
        ph["estimate"] = t3 - t2
        if cfg["kind"] == "action":
            parallel.sharded_action(g, mc.EXPONENTIAL, None, wcfg)
        ph["estimate again"] = t() - t3
        t3 = t()
        from paper_2308_01037_b200.device import to_host
        host = to_host(y)
        t4 = t()
        ph["d2h"] = t4 - t3
        g.close()
        t5 = t()
        ph["close"] = t5 - t4
        t6 = t()
        g2 = DeviceGraph(a, gamma=beta)
        t7 = t()
        ph["DeviceGraph(host a)"] = t7 - t6
        g2.close()
        print(f"rep {rep}: " + "  ".join(f"{k}={v * 1e3:.2f}ms" for k, v in ph.items()), flush=True)
    assert host.shape == (a.n,)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
