"""e2e pipeline variants at cfg2 with the real kernel (ts_marginals on device staging, argument
marshalling hoisted): copy-in on a side stream into NS staging buffers, kernel + copy-back on
the main stream; NS = 2 (the library's pipeline) vs 3; with / without the two tiny copies."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, N, E, C = cfg.B, cfg.N, cfg.E, cfg.C
L = tsb._lib.load()
G = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gather2.so"))
hp = tsb.host_empty((B, E, C, C)); hp.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hm = tsb.host_empty((B, E, C, C)); hl = tsb.host_empty((B,)); hf = tsb.host_empty((B,), torch.int32)
st = torch.cuda.current_stream(dev); cin = torch.cuda.Stream(dev); side = torch.cuda.Stream(dev)
ws = tsb.Workspace(dev)
def run(NS, tiny, n_it=400):
    dp = [torch.empty((B, E, C, C), device=dev) for _ in range(NS)]
    dm = torch.empty((B, E, C, C), device=dev); dl = torch.empty(B, device=dev); df = torch.empty(B, dtype=torch.int32, device=dev)
    chains = [tsb._lib.ts_chain(B, N, C, p.data_ptr(), None) for p in dp]
    need = int(L.ts_workspace_bytes(ctypes.byref(chains[0]), tsb._lib.TS_OP_MARG, tsb._lib.TS_LOG)); wp = ws.ptr(need)
    done = [None] * NS
    def one(k):
        p = k % NS
        if done[p] is not None: cin.wait_event(done[p])
        with torch.cuda.stream(cin):
            dp[p].copy_(hp, non_blocking=True); ev = torch.cuda.Event(); ev.record(cin)
        st.wait_event(ev)
        if tiny == "mapped":  # the kernel stores logZ / flags straight into the pinned host buffers
            L.ts_marginals(ctypes.byref(chains[p]), tsb._lib.TS_LOG, dm.data_ptr(), hl.data_ptr(), hf.data_ptr(), wp, need, st.cuda_stream)
        else:
            L.ts_marginals(ctypes.byref(chains[p]), tsb._lib.TS_LOG, dm.data_ptr(), dl.data_ptr(), df.data_ptr(), wp, need, st.cuda_stream)
        if tiny == "gather":  # one 1-warp kernel stores logZ / flags into the pinned host buffers
            hm.copy_(dm, non_blocking=True)
            G.gather2_launch(ctypes.c_void_p(hl.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                             ctypes.c_void_p(hf.data_ptr()), ctypes.c_void_p(df.data_ptr()), B,
                             ctypes.c_void_p(st.cuda_stream))
        elif tiny == "side":  # the two small copies on a forked stream, beside the big one
            side.wait_stream(st)
            with torch.cuda.stream(side):
                hl.copy_(dl, non_blocking=True); hf.copy_(df, non_blocking=True)
            hm.copy_(dm, non_blocking=True)
            st.wait_stream(side)
        elif tiny == "first":  # small copies before the big one
            hl.copy_(dl, non_blocking=True); hf.copy_(df, non_blocking=True)
            hm.copy_(dm, non_blocking=True)
        else:
            hm.copy_(dm, non_blocking=True)
            if tiny:
                hl.copy_(dl, non_blocking=True); hf.copy_(df, non_blocking=True)
        e = torch.cuda.Event(); e.record(st); done[p] = e
    t0 = time.perf_counter(); k = 0
    while time.perf_counter() - t0 < 0.1:
        one(k); k += 1
        if k % 32 == 0: torch.cuda.synchronize()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(n_it): one(k + i)
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n_it * 1e3
for r in range(2):
    for NS in (2,):
        for tiny in (True, False, "gather"):
            print(f"NS={NS} tiny_copies={tiny}: {run(NS, tiny):.1f} us/call", flush=True)
f = lambda: tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws)
for _ in range(200): f()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(400): f()
e1.record(); torch.cuda.synchronize(); print(f"library marginals_host: {e0.elapsed_time(e1) / 400 * 1e3:.1f} us/call")
