import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import paper_2002_00876_b200 as tsb, tsgen
cfg = tsgen.CONFIGS[5]
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, cfg)
out = torch.empty_like(pot)
def t(fn, n=5):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[n // 2]
for L in (0, 1772, 1200, 886, 600, 443):
    tsb.set_plan_chunk(L)
    ms = t(lambda: tsb.marginals(pot, out=out))
    print(json.dumps({"L": L, "ms": round(ms, 3), "launches": tsb.last_launch_count()}), flush=True)
tsb.set_plan_chunk(0)
