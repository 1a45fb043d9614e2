#!/usr/bin/env python
"""Calibrate the Viterbi plan choice (abi.cu vit_chunk): for each BxNxC shape, time the serial
sweep (plan_chunk 0 before the auto rule) and the time-chunked max-plus scan (vchunk.cu) at
chunk lengths giving B*P = 148, 296, 592 chunks.  Device-resident tsgen inputs, CUDA events,
median of --iters.  JSON lines on stdout."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402
from plan_calib import time_call  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--segs", default="148,296,592")
    ap.add_argument("--shapes", default="1x65536x128,4x65536x128,16x16384x128,64x4096x128,"
                    "1x65536x64,4x65536x64,16x16384x64,64x8192x64,"
                    "1x65536x32,4x65536x32,16x16384x32,64x8192x32")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for sh in args.shapes.split(","):
        B, N, C = [int(x) for x in sh.split("x")]
        E = N - 1
        pot = torch.empty((B, E, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, 1234)
        runs = [("serial", -1)]
        for nseg in [int(x) for x in args.segs.split(",")]:
            P = max(1, nseg // B)
            L = (E + P - 1) // P
            if P >= 2 and L >= 2:
                runs.append((f"segs{B * P}", L))
        ref = None
        for name, L in runs:
            tsb.set_plan_chunk(L if L > 0 else E)  # L = E: one chunk -> the serial sweep
            ms = time_call(lambda: tsb.viterbi(pot), 1, args.iters)
            path, score, _ = tsb.viterbi(pot)
            same = None
            if ref is None:
                ref = (path.clone(), score.clone())
            else:
                same = bool(torch.equal(ref[0], path) and torch.equal(ref[1], score))
            print(json.dumps({"B": B, "N": N, "C": C, "variant": name, "chunk": L,
                              "kernel": tsb.last_kernel(), "ms": round(ms, 4),
                              "same_as_serial": same}), flush=True)
        tsb.set_plan_chunk(0)
        del pot
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
