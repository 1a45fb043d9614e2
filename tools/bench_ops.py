#!/usr/bin/env python
"""Side measurements of the SURVEY §8(f) entry points (entropy, log_prob, sampling, K-best,
semi-Markov) and of time-sharded virtual segments on one B200 (not the bench.py contract).
Device-resident seeded inputs, CUDA events, median of `--iters` calls after warm-up."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_00876_b200 as tsb  # noqa: E402
import tsgen  # noqa: E402


def timeit(fn, warmup=3, iters=10):
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
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for no in (2, 3):
        cfg = tsgen.CONFIGS[no]
        pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, cfg)
        tok = cfg.B * cfg.N
        z = torch.zeros((cfg.B, cfg.N), dtype=torch.int32, device=dev)
        u = torch.rand((4, cfg.B, cfg.N), device=dev)
        out = torch.empty_like(pot)
        for name, fn in [("marginals", lambda: tsb.marginals(pot, out=out)),
                         ("entropy", lambda: tsb.entropy(pot, out=out)),
                         ("expectation", lambda: tsb.expectation(pot, pot, out=out)),
                         ("log_prob", lambda: tsb.log_prob(pot, z)),
                         ("sample_k4", lambda: tsb.sample(pot, u)),
                         ("kbest_k4", lambda: tsb.kbest(pot, 4)),
                         ("viterbi", lambda: tsb.viterbi(pot))]:
            ms = timeit(fn, iters=args.iters)
            rows.append({"config": f"cfg{no}", "op": name, "ms": ms, "tokens_per_s": tok / (ms / 1e3)})
        del pot, out
        torch.cuda.empty_cache()
    # semi-Markov at the Table-1 shape with K = 4
    sm = torch.from_numpy(np.random.default_rng(0).standard_normal((32, 24, 4, 20, 20)).astype(
        np.float32)).to(dev)
    ms = timeit(lambda: tsb.semimarkov(sm), iters=args.iters)
    rows.append({"config": "semi B32 N25 K4 C20", "op": "semimarkov", "ms": ms,
                 "tokens_per_s": 32 * 25 / (ms / 1e3)})
    ms = timeit(lambda: tsb.semimarkov_viterbi(sm), iters=args.iters)
    rows.append({"config": "semi B32 N25 K4 C20", "op": "semimarkov_viterbi", "ms": ms,
                 "tokens_per_s": 32 * 25 / (ms / 1e3)})
    # wide-label log path (128 < C <= 256: exact SIMT fallback), cfg4's shape
    cfg = tsgen.CONFIGS[4]
    pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, cfg)
    out = torch.empty_like(pot)
    ms = timeit(lambda: tsb.marginals(pot, out=out), warmup=1, iters=3)
    rows.append({"config": "cfg4 shape (log)", "op": "marginals", "ms": ms,
                 "tokens_per_s": cfg.B * cfg.N / (ms / 1e3), "kernel": tsb.last_kernel(),
                 "hbm_frac": 2 * cfg.B * cfg.E * cfg.C * cfg.C * 4 / (ms / 1e3) / 6550e9})
    for r in rows:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
