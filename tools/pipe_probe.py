"""Steady-state period of the e2e copy pipeline pattern (after a PCIe warm-up): raw
H2D/D2H on two streams with double-buffered staging, vs ts_marginals_host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, E, C = cfg.B, cfg.E, cfg.C
n = B * E * C * C
hp = tsb.host_empty((n,)); hm = tsb.host_empty((n,))
dpot = [torch.empty(n, device=dev) for _ in range(2)]
dm = torch.empty(n, device=dev)
cin, st = torch.cuda.Stream(), torch.cuda.current_stream()
def timed(fn, n_it):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(n_it): fn(k)
    e1.record(st); torch.cuda.synchronize(); return e0.elapsed_time(e1) / n_it * 1e3
warm = lambda k: dpot[0].copy_(hp, non_blocking=True)
for _ in range(20): timed(warm, 50)   # PCIe ramp-up (~30 ms of traffic)
print("H2D alone:", round(timed(warm, 200), 1))
print("D2H alone:", round(timed(lambda k: hm.copy_(dm, non_blocking=True), 200), 1))
done = [None, None]
def pipe(k, kernel=False):
    p = k & 1
    if done[p] is not None: cin.wait_event(done[p])
    with torch.cuda.stream(cin):
        dpot[p].copy_(hp, non_blocking=True)
        ev = torch.cuda.Event(); ev.record(cin)
    st.wait_event(ev)
    if kernel: dm.copy_(dpot[p])      # stand-in device work (~1 us)
    hm.copy_(dm, non_blocking=True)
    e = torch.cuda.Event(); e.record(st); done[p] = e
print("pipelined H2D(k+1) || D2H(k):", round(timed(pipe, 300), 1))
dl = torch.empty(B, device=dev); hl0 = tsb.host_empty((B,)); hf0 = tsb.host_empty((B,))
dmg = torch.empty((B, E, C, C), device=dev)
def pipe2(k, tiny=False, kern=False):
    p = k & 1
    if done[p] is not None: cin.wait_event(done[p])
    with torch.cuda.stream(cin):
        dpot[p].copy_(hp, non_blocking=True)
        ev = torch.cuda.Event(); ev.record(cin)
    st.wait_event(ev)
    if kern:
        m, lz, fl = tsb.marginals(dpot[p].view(B, E, C, C))
        hm.copy_(m.view(-1), non_blocking=True)
    else:
        hm.copy_(dm, non_blocking=True)
    if tiny:
        hl0.copy_(dl, non_blocking=True); hf0.copy_(dl, non_blocking=True)
    e = torch.cuda.Event(); e.record(st); done[p] = e
done[0] = done[1] = None
print("pipelined + 2 tiny D2H:", round(timed(lambda k: pipe2(k, True), 300), 1))
done[0] = done[1] = None
print("pipelined + kernel (tsb.marginals):", round(timed(lambda k: pipe2(k, False, True), 300), 1))
done[0] = done[1] = None
print("pipelined + kernel + 2 tiny D2H:", round(timed(lambda k: pipe2(k, True, True), 300), 1))
print("same, both on one stream:", round(timed(lambda k: (dpot[0].copy_(hp, non_blocking=True), hm.copy_(dm, non_blocking=True)), 300), 1))
h = tsb.host_empty((B, E, C, C)); h.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hmm = tsb.host_empty((B, E, C, C)); hl = tsb.host_empty((B,)); hf = tsb.host_empty((B,), torch.int32)
ws = tsb.Workspace(dev)
f = lambda k: tsb.marginals_host(h, hmm, hl, hf, device=dev, ws=ws)
for _ in range(5): timed(f, 50)
print("marginals_host:", round(timed(f, 300), 1))
tsb.set_host_pipeline(False)
for _ in range(2): timed(f, 50)
print("marginals_host, no pipeline:", round(timed(f, 300), 1))
tsb.set_host_pipeline(True)
