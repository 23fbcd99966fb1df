import sys, math, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2308_01037_b200 as mc
from tests.test_gpu_configs import _masked_target
for name, cfg in [("ba400-like", None), ("config2", bench.CONFIGS[2])]:
    if cfg is None:
        from tests import golden_io
        from scipy import sparse
        c = golden_io.load('ba400'); a0 = c.sa
        A = sparse.csr_array((a0.vals, a0.col_ids, a0.row_ptr), shape=(a0.n, a0.n))
        lam = abs(np.linalg.eigvalsh(A.toarray())).max()
        class M: pass
        m = M(); m.csr = A; m.csc = A.tocsc(); m.symmetric_hint = True
        g = mc.DeviceGraph(m, gamma=1/lam); n_walks = 300; ms = 28
    else:
        a, beta, n_walks = bench.make_graph(cfg); g = mc.DeviceGraph(a, gamma=beta); ms = cfg["max_steps"]
    zeta = mc.EXPONENTIAL.prefix(ms + 2)
    for path in ("funm", "walk_action"):
        R = 64
        ys = torch.empty((R, g.n), dtype=torch.float64, device="cuda")
        for s in range(R):
            wc = mc.WalkConfig(n_walks, 1e-300, ms, 100 + s)
            if path == "funm":
                res = mc.rand_funm_action(g, mc.EXPONENTIAL, None, wc, as_tensor=True)
            else:
                ni0, pre0 = g.allocate(n_walks)
                res = mc.rand_funm_action(g, mc.EXPONENTIAL, torch.ones(g.n, dtype=torch.float64, device="cuda"), wc,
                                          budgets=ni0.cpu().numpy(), as_tensor=True)
            ys[s] = res.values
        ni = res.aux["ni"]
        tgt = _masked_target(g, zeta, ms, ni)
        mean = ys.mean(0); se = ys.std(0) / math.sqrt(R)
        ok = se > 0
        z = ((mean - tgt)[ok] / se[ok]).cpu().numpy()
        print(name, path, "frac0", float((ni == 0).double().mean()), "z mean", z.mean(), "sd", z.std(), "max", np.abs(z).max(),
              "frac3", np.mean(np.abs(z) <= 3), flush=True)
        bad = torch.nonzero(ok).flatten()[torch.from_numpy(np.argsort(-np.abs(z))[:5]).cuda()]
        deg = (g.row_ptr[1:] - g.row_ptr[:-1])
        print("  worst nodes", bad.tolist(), "deg", deg[bad].tolist(), "ni", ni[bad].tolist(), "mean", mean[bad].tolist(), "tgt", tgt[bad].tolist())
