"""One K-best Viterbi call at the cfg3 shape (B=256, N=512, C=64) for ncu; timed with CUDA
events when run without a profiler (median of 5 after a warm-up).  argv: [K] [sample]"""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00876_b200 as tsb, tsgen
K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = tsgen.CONFIGS[3]
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, cfg)
fns = {"kbest": lambda: tsb.kbest(pot, K)}
if len(sys.argv) > 2:
    noise = torch.rand((K, cfg.B, cfg.N), device="cuda:0")
    fns["sample"] = lambda: tsb.sample(pot, noise)
for name, fn in fns.items():
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"op": name, "K": K, "shape": [cfg.B, cfg.N, cfg.C], "kernel": tsb.last_kernel(),
                      "ms_median": sorted(ts)[2]}), flush=True)
