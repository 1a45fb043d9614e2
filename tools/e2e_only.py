"""e2e leg only: steady-state us/call of ts_marginals_host at cfg2 (after a 60 ms warm-up)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, E, C = cfg.B, cfg.E, cfg.C
h = tsb.host_empty((B, E, C, C)); h.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hm = tsb.host_empty((B, E, C, C)); hl = tsb.host_empty((B,)); hf = tsb.host_empty((B,), torch.int32)
ws = tsb.Workspace(dev)
f = lambda: tsb.marginals_host(h, hm, hl, hf, device=dev, ws=ws)
t0 = time.perf_counter(); n = 0
while time.perf_counter() - t0 < 0.1:
    f(); n += 1
    if n % 32 == 0: torch.cuda.synchronize()
torch.cuda.synchronize()
res = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(400): f()
    e1.record(); torch.cuda.synchronize(); res.append(e0.elapsed_time(e1) / 400 * 1e3)
print("us/call:", [round(x, 1) for x in res], "warm calls", n)
