"""Semi-Markov timing (f4): the expanded-state scan at N = 4097 (auto plan) and, at N = 255
(E < 256: the auto plan keeps the segmental one-CTA kernel), both plans side by side."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2002_00876_b200 as tsb
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(it):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]
rng = np.random.default_rng(0)
for (B, N, K, C, L) in [(8, 4097, 4, 20, 0), (8, 255, 4, 20, 0), (8, 255, 4, 20, 16), (32, 255, 4, 20, 0), (32, 255, 4, 20, 16)]:
    pot = torch.from_numpy((rng.integers(-128, 129, size=(B, N - 1, K, C, C)) / 256.0).astype(np.float32)).cuda()
    tsb.set_plan_chunk(L)
    ms = t(lambda: tsb.semimarkov(pot))
    k1 = tsb.last_kernel()
    msv = t(lambda: tsb.semimarkov_viterbi(pot))
    print(json.dumps({"B": B, "N": N, "K": K, "C": C, "plan_chunk": L, "marginals_ms": ms, "kernel": k1,
                      "viterbi_ms": msv, "viterbi_kernel": tsb.last_kernel(), "tokens_per_s": B * N / ms * 1e3}), flush=True)
    del pot
tsb.set_plan_chunk(0)
