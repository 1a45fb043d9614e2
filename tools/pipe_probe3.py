"""Three-stage e2e pipeline probe at cfg2 (copy-in, kernel, copy-back each on its own stream,
double-buffered staging for inputs and outputs) vs the two-stream pipeline the library runs."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, N, E, C = cfg.B, cfg.N, cfg.E, cfg.C
nel = B * E * C * C
L = tsb._lib.load()
hp = tsb.host_empty((B, E, C, C)); hp.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hout = tsb.host_empty((nel + 2 * B,))
st = torch.cuda.current_stream(dev)
cin, ck, cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
ws = tsb.Workspace(dev)
dp = [torch.empty((B, E, C, C), device=dev) for _ in range(2)]
do = [torch.empty(nel + 2 * B, device=dev) for _ in range(2)]
ch = [tsb._lib.ts_chain(B, N, C, p.data_ptr(), None) for p in dp]
need = int(L.ts_workspace_bytes(ctypes.byref(ch[0]), tsb._lib.TS_OP_MARG, tsb._lib.TS_LOG)); wp = ws.ptr(need)
kdone = [None, None]; odone = [None, None]
def one(k):
    p = k % 2
    if kdone[p] is not None: cin.wait_event(kdone[p])
    with torch.cuda.stream(cin):
        dp[p].copy_(hp, non_blocking=True); ein = torch.cuda.Event(); ein.record(cin)
    ck.wait_event(ein)
    if odone[p] is not None: ck.wait_event(odone[p])
    base = do[p].data_ptr()
    L.ts_marginals(ctypes.byref(ch[p]), tsb._lib.TS_LOG, base, base + 4 * nel, base + 4 * (nel + B), wp, need, ck.cuda_stream)
    ek = torch.cuda.Event(); ek.record(ck); kdone[p] = ek
    cout.wait_event(ek)
    with torch.cuda.stream(cout):
        hout.copy_(do[p], non_blocking=True); eo = torch.cuda.Event(); eo.record(cout)
    odone[p] = eo
    st.wait_event(eo)
def bench(fn, n=400):
    t0 = time.perf_counter(); k = 0
    while time.perf_counter() - t0 < 0.1:
        fn(k); k += 1
        if k % 32 == 0: torch.cuda.synchronize()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(n): fn(k + i)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
hm = hout[:nel].view(B, E, C, C); hl = hout[nel:nel + B]; hf = hout[nel + B:].view(torch.int32)
for r in range(3):
    print(f"three-stage: {bench(one):.1f} us/call", flush=True)
    print(f"library ts_marginals_host: {bench(lambda k: tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws)):.1f} us/call", flush=True)
