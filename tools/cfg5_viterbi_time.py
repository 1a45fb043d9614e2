"""cfg5 (B=4, N=65536, C=128) Viterbi on one GPU: the serial sweeps (vit2 cluster split, one CTA;
plan chunk >= N forces the serial plan), the default auto plan, and the time-chunked max-plus
scan (vchunk.cu) at a few chunk lengths.  CUDA events, one
timed call after a warm-up call per variant."""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_00876_b200 as tsb, tsgen
cfg = tsgen.CONFIGS[5]
pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, cfg)
def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
ref = None
for name, vs, L in [("serial vit2", 0, cfg.N), ("auto plan", 0, 0), ("serial one-CTA", -1, cfg.N),
                    ("chunked L=512", 0, 512), ("chunked L=1772", 0, 1772), ("chunked L=4096", 0, 4096)]:
    tsb.set_viterbi_split(vs); tsb.set_plan_chunk(L)
    ms = t(lambda: tsb.viterbi(pot))
    path, score, flags = tsb.viterbi(pot)
    same = None
    if ref is None: ref = (path.clone(), score.clone())
    else: same = bool(torch.equal(ref[0], path) and torch.equal(ref[1], score))
    print(json.dumps({"config": "cfg5 viterbi", "variant": name, "kernel": tsb.last_kernel(),
                      "ms": ms, "tokens_per_s": cfg.B * cfg.N / ms * 1e3, "same_as_serial": same}), flush=True)
tsb.set_viterbi_split(0); tsb.set_plan_chunk(0)
