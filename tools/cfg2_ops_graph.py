"""cfg2 ops in a CUDA graph of 500 back-to-back calls (device-resident, L2-warm): marginals vs
logZ only vs entropy — the per-call cost without host launch overhead."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00876_b200 as tsb, tsgen
cfg = tsgen.CONFIGS[2]
dev = torch.device("cuda:0")
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
tsgen.fill_torch(pot, cfg)
ws = tsb.Workspace(dev)
marg = torch.empty_like(pot)
def graph_time(fn, n=500):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for name, fn in [("marginals", lambda: tsb.marginals(pot, ws=ws, out=marg)),
                 ("logz", lambda: tsb.logpartition(pot, ws=ws)),
                 ("entropy", lambda: tsb.entropy(pot, out=marg))]:
    print(json.dumps({"op": name, "us_per_call": graph_time(fn)}), flush=True)
for N in (1, 2, 5, 13, 25):
    p = torch.empty((cfg.B, max(N - 1, 1), cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(p, 7)
    if N == 1:
        p = p[:, :0].contiguous()
    m = torch.empty_like(p)
    print(json.dumps({"op": "marginals", "N": N, "us_per_call": graph_time(lambda: tsb.marginals(p, ws=ws, out=m)),
                      "kernel": tsb.last_kernel()}), flush=True)
