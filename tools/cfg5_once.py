import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2002_00876_b200 as tsb, tsgen
cfg = tsgen.CONFIGS[5]
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, cfg)
out = torch.empty_like(pot)
for _ in range(2): tsb.marginals(pot, out=out)
torch.cuda.synchronize()
