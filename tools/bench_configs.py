#!/usr/bin/env python
"""Side measurements on one B200 for every BASELINE config (not the bench.py contract line).

Device-resident inputs (tsgen device fill), CUDA events on the current stream, warm-up
calls first; cfg3..5 inputs exceed the 126 MB L2 so every call streams from HBM.
Prints one JSON line per config with time, tokens/s and the HBM roofline fraction of the
algorithmic bytes (logZ+marginals: read l + write mu = 8 C^2 B/edge; Viterbi: 4 C^2 B/edge).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def time_call(fn, warmup, iters):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(iters):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    return times[len(times) // 2], times[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--tc", type=int, default=3, help="leaf summaries: 3 3xTF32, 1 1xTF32, 0 SIMT")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = peak_gbs()
    tsb.set_plan_chunk(args.chunk)
    tsb.set_tc_summary(args.tc)
    for no in [int(x) for x in args.configs.split(",")]:
        cfg = tsgen.CONFIGS[no]
        B, N, C, E = cfg.B, cfg.N, cfg.C, cfg.E
        pot = torch.empty((B, E, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, cfg)
        if cfg.op == "viterbi":
            fn = lambda: tsb.viterbi(pot)  # noqa: E731
            alg = 4 * C * C * B * E
        else:
            out = torch.empty_like(pot)
            fn = lambda: tsb.marginals(pot, out=out)  # noqa: E731
            alg = 8 * C * C * B * E
        med, best = time_call(fn, 2, args.iters)
        launches = tsb.last_launch_count()
        gbs = alg / (med / 1e3) / 1e9
        print(json.dumps({"config": f"cfg{no}", "op": cfg.op, "B": B, "N": N, "C": C,
                          "ms_median": med, "ms_best": best, "tokens_per_s": B * N / (med / 1e3),
                          "alg_bytes": alg, "achieved_gbs": gbs, "frac_hbm": gbs / peak,
                          "launches": launches, "plan_chunk": args.chunk, "tc": args.tc}), flush=True)
        del pot
        if cfg.op != "viterbi":
            del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
