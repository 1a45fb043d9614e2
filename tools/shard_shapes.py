#!/usr/bin/env python
"""Per-rank shapes of the batch-sharded BASELINE configs on one B200 (verdict r1 item 4).

With batch sharding over G GPUs each rank runs the same kernel on B/G sequences, so the
scaling efficiency at G is T(B) / (G * T(B/G)) with T measured on one GPU (no collective on
the data path).  For each per-rank batch this times the auto plan and the alternatives the
plan could pick (cfg3: P = 1 meet-in-the-middle vs the chunked scan; cfg4: the vit2 cluster
split sizes).  Device-resident inputs larger than L2 (>= 268 MB), CUDA events, median of
`--iters` calls after warm-up; nvidia-smi SM clock sampled after each shape.  One JSON line
per (config, B, variant) on stdout.
"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
        sm, mx, reasons = [x.strip() for x in out.strip().split("\n")[0].split(",")]
        return {"sm_mhz": float(sm), "sm_max_mhz": float(mx), "throttle": reasons}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


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
    ap.add_argument("--iters", type=int, default=9)
    ap.add_argument("--configs", default="3,4")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for no in [int(x) for x in args.configs.split(",")]:
        cfg = tsgen.CONFIGS[no]
        Bfull = cfg.B
        pot_full = torch.empty((Bfull, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot_full, cfg)
        for G in (1, 2, 4, 8):
            B = Bfull // G
            pot = pot_full[:B]
            if cfg.op == "viterbi":
                variants = [("auto", 0), ("one_cta", -1)] + [(f"cluster{g}", g) for g in (1, 2, 4, 8)]
                for name, knob in variants:
                    tsb.set_viterbi_split(knob)
                    fn = lambda: tsb.viterbi(pot)  # noqa: E731
                    ms = time_call(fn, 3, args.iters)
                    print(json.dumps({"config": no, "op": "viterbi", "ranks": G, "B_per_rank": B,
                                      "variant": name, "kernel": tsb.last_kernel(), "ms": ms,
                                      "tokens_per_s_per_rank": B * cfg.N / ms * 1e3, "clocks": clocks()}),
                          flush=True)
                tsb.set_viterbi_split(0)
            else:
                for name, chunk in [("auto", 0), ("serial_P1", cfg.E)]:
                    tsb.set_plan_chunk(chunk)
                    fn = lambda: tsb.marginals(pot)  # noqa: E731
                    ms = time_call(fn, 3, args.iters)
                    print(json.dumps({"config": no, "op": "marginals", "ranks": G, "B_per_rank": B,
                                      "variant": name, "kernel": tsb.last_kernel(),
                                      "launches": tsb.last_launch_count(), "ms": ms,
                                      "tokens_per_s_per_rank": B * cfg.N / ms * 1e3, "clocks": clocks()}),
                          flush=True)
                tsb.set_plan_chunk(0)
        del pot_full
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
