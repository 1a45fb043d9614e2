"""Does the H2D rate of a 1.2 MB pinned payload depend on warm-up / idle time?  Batches of
copies timed back to back, then after idle gaps; also the e2e entry point per batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
hp = torch.ones(1228800 // 4).pin_memory(); d = torch.empty_like(hp, device=dev)
def batch(fn, n=50):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n * 1e3
cp = lambda: d.copy_(hp, non_blocking=True)
print("H2D batches of 50 (us/copy):", [round(batch(cp), 1) for _ in range(12)])
for gap in (0.001, 0.01, 0.1, 1.0):
    time.sleep(gap)
    print(f"after {gap}s idle:", [round(batch(cp, 10), 1) for _ in range(4)])
cfg = tsgen.CONFIGS[2]
B, E, C = cfg.B, cfg.E, cfg.C
h = tsb.host_empty((B, E, C, C)); h.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hm = tsb.host_empty((B, E, C, C)); hl = tsb.host_empty((B,)); hf = tsb.host_empty((B,), torch.int32)
ws = tsb.Workspace(dev)
f = lambda: tsb.marginals_host(h, hm, hl, hf, device=dev, ws=ws)
print("marginals_host batches of 50 (us/call):", [round(batch(f), 1) for _ in range(12)])
time.sleep(0.5)
print("after 0.5 s idle:", [round(batch(f, 20), 1) for _ in range(6)])
