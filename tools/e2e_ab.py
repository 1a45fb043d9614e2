#!/usr/bin/env python
"""A/B of the host-buffer entry point (ts_marginals_host) with different library builds
(debug tool): python tools/e2e_ab.py <libpath>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_00876_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402

dev = torch.device("cuda:0")
cfg = tsgen.CONFIGS[2]
B, N, C, E = cfg.B, cfg.N, cfg.C, cfg.E
hp = tsb.host_empty((B, E, C, C))
hp.copy_(torch.from_numpy(tsgen.config_potentials(cfg)))
hm = tsb.host_empty((B, E, C, C))
hl = tsb.host_empty((B,))
hf = tsb.host_empty((B,), torch.int32)
ws = tsb.Workspace(dev)
for _ in range(5):
    tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 400
e0.record()
for _ in range(n):
    tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=ws)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'default'}: {us:.1f} us/step, "
      f"{B * N / (us * 1e-6) / 1e6:.2f} M tok/s")
