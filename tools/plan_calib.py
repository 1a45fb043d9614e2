#!/usr/bin/env python
"""Calibrate the log-semiring plan choice (abi.cu log_plan): for each shape, time the auto plan,
the serial plan (P = 1: meet64 / fwd2+bwd2) and chunked plans with a few chunk lengths.
Device-resident tsgen inputs, CUDA events, median of --iters.  JSON lines on stdout."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402


def time_call(fn, warmup, iters):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--tc", type=int, default=3)
    ap.add_argument("--chunks", default="0,E,32,64,128,256,512,1024")
    ap.add_argument("--shapes", default="4x4096x64,8x4096x64,16x2048x64,32x1024x64,64x512x64,4x16384x64,"
                    "4x4096x32,16x2048x32,4x4096x128,16x2048x128,32x1024x128,64x1024x128")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    tsb.set_tc_summary(args.tc)
    for sh in args.shapes.split(","):
        B, N, C = [int(x) for x in sh.split("x")]
        E = N - 1
        pot = torch.empty((B, E, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, 1234, s=10)
        for L in [E if x == "E" else int(x) for x in args.chunks.split(",")]:
            if L > E:
                continue
            tsb.set_plan_chunk(L)
            ms = time_call(lambda: tsb.marginals(pot), 2, args.iters)
            print(json.dumps({"B": B, "N": N, "C": C, "chunk": L, "tc": args.tc, "kernel": tsb.last_kernel(),
                              "launches": tsb.last_launch_count(), "ms": round(ms, 4)}), flush=True)
        tsb.set_plan_chunk(0)
        del pot
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
