import sys, torch
sys.path.insert(0, "/root/repo")
import bench, paper_2308_01037_b200 as mc
from paper_2308_01037_b200 import parallel, _native
from paper_2308_01037_b200.device import DeviceGraph, WalkParams
cfg = bench.CONFIGS[2]
a, beta, n_walks = bench.make_graph(cfg)
g = DeviceGraph(a, gamma=beta)
w = mc.WalkConfig(n_walks, cfg["cutoff"], cfg["max_steps"], cfg["seed"])
p = WalkParams(w, mc.EXPONENTIAL.prefix(30))
for _ in range(3): parallel.sharded_action(g, mc.EXPONENTIAL, None, w, params=p)
torch.cuda.synchronize(); g.kernel_times(reset=True)
p.c.flags = _native.MCF_FLAG_TIME_KERNELS
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s): parallel.sharded_action(g, mc.EXPONENTIAL, None, w, params=p)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize(); g.kernel_times(reset=True)
G = torch.cuda.CUDAGraph()
with torch.cuda.graph(G): parallel.sharded_action(g, mc.EXPONENTIAL, None, w, params=p)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(8):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); G.replay(); e1.record(); torch.cuda.synchronize(); tot = e0.elapsed_time(e1)
    wm, qm, k = g.kernel_times(reset=False)
    print(f"step {tot*1e3:.1f} us  pre-walk {qm*1e3:.1f} us  walk {wm*1e3:.1f} us  post-walk {(tot - qm - wm)*1e3:.1f} us (k={k})")
