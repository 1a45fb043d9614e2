"""ts_sample timing (FFBS, K samples) at the cfg3 shape and C=128 / cfg2 shapes, with the
forward filter alone (ts_logpartition) beside it.  TS_B200_LIB selects a variant build."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n
for (B, N, C, K) in [(256, 512, 64, 4), (256, 512, 64, 32), (64, 1024, 128, 4), (32, 25, 20, 4)]:
    pot = torch.empty((B, N - 1, C, C), device=dev); tsgen.fill_torch(pot, 7, 0)
    u = torch.rand((K, B, N), device=dev)
    res = {"B": B, "N": N, "C": C, "K": K}
    res["sample_ms"] = round(t(lambda: tsb.sample(pot, u)), 4)
    res["kernel"] = tsb.last_kernel()
    res["logpartition_ms"] = round(t(lambda: tsb.logpartition(pot)), 4)
    print(json.dumps(res))
