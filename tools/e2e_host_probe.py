"""e2e leg as bench.py runs it (contiguous outputs, three-stage pipeline): host enqueue time
per call and device time per call, over repeated 400-call regions after a 60 ms warm-up."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2002_00876_b200 as tsb
import tsgen
dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, E, C = cfg.B, cfg.E, cfg.C
nel = B * E * C * C
hp = tsb.host_empty((B, E, C, C)); hp.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hout = tsb.host_empty((nel + 2 * B,))
hm, hl, hf = hout[:nel].view(B, E, C, C), hout[nel:nel + B], hout[nel + B:].view(torch.int32)
ws = tsb.Workspace(dev)
st = torch.cuda.current_stream(dev)
f = lambda: tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws)
t0 = time.perf_counter(); n = 0
while time.perf_counter() - t0 < 0.06 or n < 50:
    f(); n += 1
    if n % 32 == 0: torch.cuda.synchronize()
torch.cuda.synchronize()
for rep in range(8):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); h0 = time.perf_counter()
    for _ in range(400): f()
    h1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize()
    print(f"rep {rep}: device {e0.elapsed_time(e1) / 400 * 1e3:.1f} us/call, host enqueue {(h1 - h0) / 400 * 1e6:.1f} us/call", flush=True)
