"""Walk-kernel rate vs graph size (BA m=4, 0.64 walks per node, max_steps 28):
where does the L2 working set stop fitting?  Prints G steps/s of k_walk_action
alone (device events), cold L2 (256 MiB write before every pass)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2308_01037_b200 as mc  # noqa: E402
from paper_2308_01037_b200 import _native, graphs, parallel  # noqa: E402
from paper_2308_01037_b200.device import DeviceGraph, WalkParams  # noqa: E402


def main(sizes):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for n in sizes:
        a = graphs.barabasi_albert(n, 4, seed=0)
        beta = 1.0 / graphs.lambda_max(a)
        g = DeviceGraph(a, gamma=beta)
        nw = int(0.64 * n)
        cfg = mc.WalkConfig(nw, 1e-300, 28, 0)
        z = mc.EXPONENTIAL.prefix(30)
        p = WalkParams(cfg, z)
        v = torch.ones(g.n, dtype=torch.float64, device=g.device)
        for _ in range(3):
            y, st = parallel.sharded_action(g, mc.EXPONENTIAL, None, cfg, params=p)
        torch.cuda.synchronize()
        g.kernel_times(reset=True)
        p.c.flags = _native.MCF_FLAG_TIME_KERNELS
        em = 0
        for _ in range(5):
            flush.zero_()
            y, st = parallel.sharded_action(g, mc.EXPONENTIAL, None, cfg, params=p)
            em += int(st[1])
        torch.cuda.synchronize()
        wms, _, k = g.kernel_times(reset=True)
        info = g.info
        print(f"n={n:>8} nnz={g.nnz:>9} tables={(32 * n + 4 * g.nnz) / 2**20:7.1f} MiB layout={info['walk_layout']} "
              f"walk {wms / k * 1e3:8.1f} us  {em / (wms / 1e3) / 1e9:6.1f} G steps/s", flush=True)
        p.c.flags = 0
        g.close()


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [125_000, 250_000, 500_000, 1_000_000, 2_000_000])
