import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2002_00876_b200 as tsb, tsgen
cfg = tsgen.CONFIGS[5]
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, cfg)
tsb.set_plan_chunk(1772)
tsb.viterbi(pot); torch.cuda.synchronize()
