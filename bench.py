#!/usr/bin/env python
"""bench.py — throughput of the linear-chain CRF hot path (logZ + marginals) on B200.

Contract: `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A step = one ts_marginals call (the whole hot path: forward scan,
explicit backward scan, marginals, logZ) over one batch of the BASELINE.json metric
workload: B=32, N=25, C=20 (Table 1 caption), synthetic seeded
dyadic potentials (tsgen).  Multi-GPU: one process per GPU, each rank its own B=32
batch (weak scaling, no data-path collective); time = max over ranks.

`--impl reference` times the fp64 CPU oracle (oracle/) on the host cores as the
reference arm (this tier has no runnable upstream implementation).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec linear-chain logZ+marginals (B=32,N=25,C=20) at 1/2/4/8 B200; % roofline"
UNIT = "tokens/s"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(kernel: str, cfg_no: int):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(f"cfg{cfg_no}", {}).get(kernel)
    return None if v is None else float(v)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def oracle_baseline(cfg, seconds: float = 8.0, max_batches: int = 2000):
    """Time the fp64 oracle (as it stands) on this host: whole cfg batches, threads across b."""
    import oracle
    import tsgen

    pot = tsgen.config_potentials(cfg)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    threads = max(1, min(cfg.B, cores))
    oracle.chain_marginals(pot, threads=threads)  # warm (library load)
    n = 0
    t0 = time.perf_counter()
    while True:
        oracle.chain_marginals(pot, threads=threads)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= max_batches:
            break
    return {"value": n * cfg.tokens / el, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{n} batches of B={cfg.B} N={cfg.N} C={cfg.C} (fp64 forward-backward + "
                      f"marginals, {el:.1f} s wall)"}


def run_reference(args):
    rank, _, world = env_rank()
    if rank != 0:
        return 0
    import oracle
    import tsgen

    cfg = tsgen.CONFIGS[args.config]
    pot = tsgen.config_potentials(cfg)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    threads = max(1, min(cfg.B, cores))
    for _ in range(args.warmup):
        oracle.chain_marginals(pot, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.chain_marginals(pot, threads=threads)
    el = time.perf_counter() - t0
    v = args.steps * cfg.tokens / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (tsgen seeded dyadic potentials)",
            "config": {"workload": f"cfg{cfg.no}: {cfg.label}", "B": cfg.B, "N": cfg.N,
                       "C": cfg.C, "parallelism": "host threads across the batch"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{args.steps} batches of B={cfg.B} N={cfg.N} C={cfg.C}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_time_sharded(args):
    """Side mode (not the driver's line): cfg5-style long chains split in TIME across the
    ranks: each rank generates its edge range in place, runs the local scan
    summary, one NCCL all_gather_into_tensor of the C x C summaries, then the combine and its
    local sweeps + marginals.  Total work is fixed as N grows ("scaling": "strong").  Time =
    max over ranks of CUDA-event time around K steps (summary + all-gather + finish)."""
    import torch

    import paper_2002_00876_b200 as tsb
    import tsgen
    from paper_2002_00876_b200 import dist as tdist

    rank, local_rank, world = env_rank()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg = tsgen.CONFIGS[args.config]
    B, N, C, E = cfg.B, cfg.N, cfg.C, cfg.E
    begin, count = tdist.shard_edges(E, world, rank)
    local = torch.empty((B, count, C, C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(local, cfg.seed, cfg.quantum, t_begin=begin, E_global=E)
    seg = tsb.Segment(local, begin, N)
    marg = None

    def step():
        nonlocal marg
        summ = seg.summary()
        gathered = tdist._all_gather(summ, None) if dist is not None else summ[None]
        marg, logz, flags = seg.finish(gathered, rank, world, True)
        return logz, flags

    for _ in range(args.warmup):
        logz, flags = step()
    torch.cuda.synchronize(dev)
    assert int(flags.abs().sum()) == 0
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local_rank)
    sampler.start()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize(dev)
    sampler.stop()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.barrier()
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item()) / args.steps
    if rank == 0:
        peak, peak_src = load_peaks()
        alg = 8 * B * E * C * C
        line = {"metric": f"tokens/sec linear-chain logZ+marginals time-sharded (cfg{cfg.no}: "
                          f"B={B},N={N},C={C})", "value": B * N / (ms / 1e3), "unit": UNIT,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (tsgen, generated in place per rank)",
                "config": {"workload": f"cfg{cfg.no}: {cfg.label}",
                           "parallelism": f"time-sharded over {world} GPU(s), one NCCL "
                                          "all_gather of C x C segment summaries per step",
                           "l2": f"inputs {alg / 2 / 1e9:.1f} GB >> L2"},
                "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9 / world,
                             "peak": peak, "unit": "GB/s (per GPU)",
                             "frac": alg / (ms / 1e3) / 1e9 / world / peak,
                             "peak_source": peak_src},
                "clocks": sampler.summary()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="graph", choices=["graph", "eager"])
    ap.add_argument("--sets", type=int, default=0, help="rotating buffer sets (0 = auto > 2x L2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--time-shard", action="store_true",
                    help="side mode: time-sharded long chains (use with --config 5)")
    ap.add_argument("--tiny-mode", type=int, default=-1,
                    help="debug: cfg2 kernel variant (ts_set_tiny: 1 default, 0 general kernel)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.time_shard:
        return run_time_sharded(args)

    import torch

    import paper_2002_00876_b200 as tsb
    import tsgen

    rank, local_rank, world = env_rank()
    if args.tiny_mode >= 0:
        tsb.set_tiny(args.tiny_mode)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    cfg = tsgen.CONFIGS[args.config]
    assert cfg.op == "marg", "bench times logZ + marginals configs"
    B, N, C, E = cfg.B, cfg.N, cfg.C, cfg.E
    set_bytes = 2 * B * E * C * C * 4
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    R = args.sets or max(2, int((2 * l2 + set_bytes - 1) // set_bytes))
    R = min(R, max(2, int(20e9 // set_bytes)))
    pots, margs = [], []
    for r in range(R):
        p = torch.empty((B, E, C, C), dtype=torch.float32, device=dev)
        # each rank/set its own batch: seed offset by (rank, set); values from the same recipe
        tsgen.fill_torch(p, cfg.seed + 1000003 * rank + r, cfg.quantum)
        pots.append(p)
        margs.append(torch.empty_like(p))
    logz = torch.empty(B, dtype=torch.float32, device=dev)
    flags = torch.empty(B, dtype=torch.int32, device=dev)
    ws = tsb.Workspace(dev)
    stream = torch.cuda.current_stream(dev)

    # a prepared ABI call per buffer set (argument marshalling hoisted out of the loop)
    import ctypes

    L = tsb._lib.load()
    chains = [tsb._lib.ts_chain(B, N, C, p.data_ptr(), None) for p in pots]
    need = int(L.ts_workspace_bytes(ctypes.byref(chains[0]), tsb._lib.TS_OP_MARG, tsb._lib.TS_LOG))
    wptr = ws.ptr(need)

    def step(k, st):
        r = k % R
        rc = L.ts_marginals(ctypes.byref(chains[r]), tsb._lib.TS_LOG, margs[r].data_ptr(),
                            logz.data_ptr(), flags.data_ptr(), wptr, need, st)
        if rc != 0:
            raise tsb.TsError(rc, "ts_marginals")

    st_handle = stream.cuda_stream
    for k in range(args.warmup):
        step(k, st_handle)
    launches_per_step = tsb.last_launch_count()
    kernel = tsb.last_kernel()
    torch.cuda.synchronize(dev)

    graph = None
    if args.mode == "graph":
        side = torch.cuda.Stream(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            h = torch.cuda.current_stream(dev).cuda_stream
            for k in range(args.steps):
                step(k, h)
        graph.replay()  # warm the instantiated graph
        torch.cuda.synchronize(dev)

    sampler = ClockSampler(local_rank) if rank == 0 or True else None
    sampler.start()
    # settle clocks under this load for ~1 s (untimed), then the timed region
    t_end = time.perf_counter() + 1.0
    k = 0
    while time.perf_counter() < t_end:
        if graph is not None:
            graph.replay()
        else:
            for _ in range(200):
                step(k, st_handle)
                k += 1
        torch.cuda.synchronize(dev)

    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for k in range(args.steps):
            step(k, st_handle)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    sampler.stop()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # end-to-end through the public C-ABI host-buffer entry point (pinned host I/O)
    e2e_steps = args.e2e_steps or max(20, min(args.steps, 400))
    # page-locked host buffers from the library allocator (ts_host_alloc)
    hp = tsb.host_empty((B, E, C, C))
    hp.copy_(pots[0].cpu())
    hm = tsb.host_empty((B, E, C, C))
    hl = tsb.host_empty((B,))
    hf = tsb.host_empty((B,), torch.int32)
    hws = tsb.Workspace(dev)
    for _ in range(3):
        tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=hws)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        tsb.marginals_host(hp, hm, hl, hf, device=dev, ws=hws)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_steps * cfg.tokens / (float(e_ms.item()) / 1e3)

    if rank == 0:
        value = world * args.steps * cfg.tokens / (ms_max / 1e3)
        peak, peak_src = load_peaks()
        alg_bytes = 8 * B * E * C * C  # read l + write mu, per launch
        # the step is one launch of a fused kernel for the short-chain plans (cfg2): its
        # average launch duration is the timed region / launches
        launch_s = (ms / 1e3) / (args.steps * launches_per_step) if launches_per_step == 1 \
            else None
        achieved = (alg_bytes / launch_s / 1e9) if launch_s else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (tsgen seeded dyadic potentials, DESIGN.md §3)",
            "config": {"workload": f"cfg{cfg.no}: {cfg.label}", "B": B, "N": N, "C": C,
                       "global_batch": B * world, "seq_len": N,
                       "parallelism": f"batch-sharded dp{world} (B={B} per GPU, no collective)",
                       "l2": f"inputs rotate over {R} buffer sets ({R * set_bytes / 1e6:.0f} MB > "
                             f"{l2 / 1e6:.0f} MB L2)",
                       "launch": "CUDA graph of K ts_marginals calls" if graph else "eager"},
            "roofline": {"bound": "hbm", "kernel": kernel,
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": load_traffic(kernel, cfg.no),
                         "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                         "launch_s": launch_s},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": B * E * C * C * 4,
                    "d2h_bytes_per_step": B * E * C * C * 4 + 8 * B,
                    "api": "ts_marginals_host (ts_host_alloc page-locked host buffers; H2D, kernels, "
                           "D2H inside every call)"},
            "gpu_launches": args.steps * launches_per_step,
            "clocks": sampler.summary(),
            "paper_context": {"value": 390000, "unit": UNIT,
                              "hw": "K80 (Google Colab), PAPER.md Table 1 P:41/P:54",
                              "note": "context only, not the target"},
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_baseline(cfg)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
