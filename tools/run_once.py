#!/usr/bin/env python
"""Run one library call on a synthetic batch (for ncu captures): --op marg|logz|viterbi."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="marg")
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--N", type=int, default=128)
ap.add_argument("--C", type=int, default=256)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--vsplit", type=int, default=0)
args = ap.parse_args()
tsb.set_viterbi_split(args.vsplit)
pot = torch.empty((args.B, args.N - 1, args.C, args.C), dtype=torch.float32, device="cuda:0")
tsgen.fill_torch(pot, 1234, tsgen.quantum(args.N - 1))
for _ in range(args.reps):
    if args.op == "viterbi":
        tsb.viterbi(pot)
    elif args.op == "logz":
        tsb.logpartition(pot)
    else:
        tsb.marginals(pot)
torch.cuda.synchronize()
print("ok")
