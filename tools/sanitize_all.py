#!/usr/bin/env python
"""Run every public entry point once at small sizes (for compute-sanitizer memcheck /
racecheck / synccheck under gpurun).  Exits non-zero if any call raises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402

dev = torch.device("cuda:0")
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
for (B, N, C) in [(3, 25, 20), (2, 9, 3), (2, 70, 64), (2, 40, 128), (2, 300, 20)]:
    pot = T(tsgen.potentials(B, N, C, seed=N + C))
    lengths = T(np.array([N] + [max(1, N // 2)] * (B - 1), np.int32))
    tsb.marginals(pot)
    tsb.marginals(pot, lengths)
    tsb.logpartition(pot)
    tsb.viterbi(pot, lengths)
    tsb.marginals(pot, semiring="max")
    tsb.entropy(pot)
    tsb.expectation(pot, pot)
    tsb.log_prob(pot, torch.zeros((B, N), dtype=torch.int32, device=dev))
    if C <= 128:
        tsb.sample(pot, torch.rand((2, B, N), device=dev))
    tsb.kbest(pot, 4, lengths)
for mode in (0, 2):
    tsb.set_tiny(mode)
    tsb.marginals(T(tsgen.potentials(4, 25, 20, seed=1)))
tsb.set_tiny(1)
tsb.set_plan_chunk(7)
tsb.marginals(T(tsgen.potentials(2, 200, 64, seed=2)))
tsb.marginals(T(tsgen.potentials(2, 150, 128, seed=3)))
tsb.set_plan_chunk(0)
tsb.viterbi(T(tsgen.potentials(2, 40, 256, seed=4)))
sm = np.random.default_rng(0).standard_normal((2, 14, 3, 20, 20)).astype(np.float32)
tsb.semimarkov(T(sm))
sm = np.random.default_rng(0).standard_normal((2, 14, 3, 100, 100)).astype(np.float32)
tsb.semimarkov(T(sm))
tsb.semimarkov_viterbi(T(sm))
sm = np.random.default_rng(0).standard_normal((2, 14, 3, 20, 20)).astype(np.float32)
tsb.semimarkov_viterbi(T(sm))
# wide labels (fb_wide: SMEM ring for C % 4 == 0, register path otherwise)
for Cw in (132, 131):
    pw = T(tsgen.potentials(2, 30, Cw, seed=Cw))
    tsb.marginals(pw, T(np.array([30, 9], np.int32)))
    tsb.logpartition(pw)
# time-sharded segments on one device
from paper_2002_00876_b200 import dist as tdist  # noqa: E402
pot = tsgen.potentials(2, 121, 20, seed=5)
segs = []
for r in range(3):
    b0, cnt = tdist.shard_edges(120, 3, r)
    segs.append((tsb.Segment(T(pot[:, b0:b0 + cnt]), b0, 121),
                 tsb.ViterbiSegment(T(pot[:, b0:b0 + cnt]), b0, 121)))
S = torch.stack([s.summary() for s, _ in segs])
for r, (s, _) in enumerate(segs):
    s.finish(S, r, 3)
V = torch.stack([v.summary() for _, v in segs])
M = torch.stack([v.maps(V, r, 3)[0] for r, (_, v) in enumerate(segs)])
for r, (_, v) in enumerate(segs):
    v.finish(M, r, 3)
torch.cuda.synchronize()
print("sanitize sweep OK")
