"""K-best timing at the cfg3 shape (B=256, N=512, C=64) and a few-sequence shape over the
lanes-per-column knob S; CUDA events, median of 5 after a warm-up.  JSON lines."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00876_b200 as tsb, tsgen
for (B, N, C) in [(256, 512, 64), (16, 512, 64), (32, 25, 20), (64, 256, 128)]:
    pot = torch.empty((B, N - 1, C, C), dtype=torch.float32, device="cuda:0")
    tsgen.fill_torch(pot, 11)
    for K in [1, 4, 16]:
        ref = None
        for S in [0, 1, 2, 4, 8]:
            tsb.set_kbest_split(S)
            fn = lambda: tsb.kbest(pot, K)
            fn(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); fn(); e1.record(); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            p, s, f = fn()
            same = None
            if ref is None: ref = (p.clone(), s.clone())
            else: same = bool(torch.equal(ref[0], p) and torch.equal(ref[1], s))
            print(json.dumps({"B": B, "N": N, "C": C, "K": K, "S": S, "ms_median": round(sorted(ts)[2], 4),
                              "same": same}), flush=True)
    tsb.set_kbest_split(0)
