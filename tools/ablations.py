#!/usr/bin/env python
"""Fig. 3-shaped ablations (Fig. 3) on one B200.

X4 (Fig. 3a, "lengths up to 500"): B = 16, C = 20, N in {32 .. 512}; logZ + marginals with
    the plan knob at L = E (serial sweeps), L = 1 (the pure Fig. 4 tree of C x C products),
    L = 16 and the auto plan; the torch broadcast-reduce forward loop (logZ, one
    logsumexp per step, P:330's N x M x O intermediate) beside it.
X6 (Fig. 3c, label sizes): B = 16, N = 20, C in {20 .. 100}; the auto plan (logZ and
    logZ + marginals) vs torch broadcast-reduce logZ and torch autograd marginals.
Device-resident tsgen inputs, CUDA events, median of --iters after warm-up; nvidia-smi SM clock
sampled per row.  One JSON line per measurement.
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


def clock():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=10).stdout.strip().split("\n")[0].split(",")
        return {"sm_mhz": float(out[0]), "throttle": out[1].strip()}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}


def timed(fn, iters, warmup=3):
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


def torch_logz(pot):
    """The paper's PyTorch baseline shape: alpha_{t+1} = logsumexp_i(alpha_t[:, i, None] + l_t)."""
    B, E, C, _ = pot.shape
    a = torch.zeros((B, C), device=pot.device, dtype=pot.dtype)
    for t in range(E):
        a = torch.logsumexp(a[:, :, None] + pot[:, t], dim=1)
    return torch.logsumexp(a, dim=1)


def torch_marg(pot):
    p = pot.detach().requires_grad_(True)
    lz = torch_logz(p)
    (g,) = torch.autograd.grad(lz.sum(), p)
    return g


def row(**kw):
    kw["clocks"] = clock()
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=9)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    # ---- X4 ----------------------------------------------------------------------------
    for N in (32, 64, 128, 256, 512):
        B, C = 16, 20
        pot = torch.empty((B, N - 1, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, 4000 + N)
        for name, L in (("serial_L=E", N - 1), ("tree_L=1", 1), ("chunk_L=16", 16), ("auto", 0)):
            tsb.set_plan_chunk(L)
            ms = timed(lambda: tsb.marginals(pot), args.iters)
            row(ablation="X4", B=B, N=N, C=C, impl=f"ts {name}", op="logZ+marginals", ms=ms,
                kernel=tsb.last_kernel(), launches=tsb.last_launch_count())
        tsb.set_plan_chunk(0)
        ms = timed(lambda: torch_logz(pot), max(3, args.iters // 3))
        row(ablation="X4", B=B, N=N, C=C, impl="torch broadcast-reduce loop", op="logZ", ms=ms)
    # ---- X6 ----------------------------------------------------------------------------
    for C in (20, 40, 60, 80, 100):
        B, N = 16, 20
        pot = torch.empty((B, N - 1, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, 6000 + C)
        ms = timed(lambda: tsb.logpartition(pot), args.iters)
        row(ablation="X6", B=B, N=N, C=C, impl="ts auto", op="logZ", ms=ms, kernel=tsb.last_kernel())
        ms = timed(lambda: tsb.marginals(pot), args.iters)
        row(ablation="X6", B=B, N=N, C=C, impl="ts auto", op="logZ+marginals", ms=ms,
            kernel=tsb.last_kernel())
        ms = timed(lambda: torch_logz(pot), args.iters)
        row(ablation="X6", B=B, N=N, C=C, impl="torch broadcast-reduce loop", op="logZ", ms=ms,
            intermediate_bytes=B * C ** 3 * 4)
        ms = timed(lambda: torch_marg(pot), args.iters)
        row(ablation="X6", B=B, N=N, C=C, impl="torch autograd", op="logZ+marginals", ms=ms)


if __name__ == "__main__":
    main()
