"""Per-call period of back-to-back overlapped fb_tiny calls (graph of K calls on rotating
buffers) vs the batch size B at N=25, C=20: capacity-bound periods scale with B."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
L = tsb._lib.load()  # TS_B200_LIB selects a variant build
N, C, E, K, R = 25, 20, 24, 1000, 160
for B in (8, 16, 32, 64, 128):
    pots = [torch.empty((B, E, C, C), device=dev) for _ in range(R)]
    for r, p in enumerate(pots): tsgen.fill_torch(p, 11 + r, 0)
    margs = [torch.empty_like(p) for p in pots]
    lz = [torch.empty(B, device=dev) for _ in range(R)]
    fl = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(R)]
    ch = [tsb._lib.ts_chain(B, N, C, p.data_ptr(), None) for p in pots]
    need = int(L.ts_workspace_bytes(ctypes.byref(ch[0]), tsb._lib.TS_OP_MARG, tsb._lib.TS_LOG))
    ws = tsb.Workspace(dev); wp = ws.ptr(need)
    def step(k, h):
        r = k % R
        L.ts_marginals(ctypes.byref(ch[r]), tsb._lib.TS_LOG, margs[r].data_ptr(), lz[r].data_ptr(), fl[r].data_ptr(), wp, need, h)
    for k in range(5): step(k, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); side = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=side):
        h = torch.cuda.current_stream().cuda_stream
        for k in range(K): step(k, h)
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / K * 1e3
    print(f"B={B:4d}: {us:.3f} us/call, {B * N / us * 1e6:.3g} tok/s", flush=True)
