"""CPU: bench.py's launch contract (no GPU needed).

`python bench.py --gpus N` outside torchrun re-launches itself with N ranks (one process per
GPU, 127.0.0.1 rendezvous) and rank 0 alone prints ONE JSON line.  Exercised through the
reference arm (the fp64 oracle on the host), which runs without a GPU.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=300):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    return lines


def test_gpus_2_spawns_ranks_and_prints_one_line():
    lines = run_bench("--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "3")
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["steps"] == 2
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["cpu"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_single_rank_reference_line():
    lines = run_bench("--impl", "reference", "--steps", "3", "--warmup", "3")
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["B"] == 32 and d["config"]["N"] == 25 and d["config"]["C"] == 20


def test_arg_defaults():
    sys.path.insert(0, ROOT)
    import bench

    a = bench.parse([])
    assert a.gpus == 1 and a.warmup >= 3 and a.side == [3, 4, 5]
    assert bench.parse(["--side", ""]).side == []
    assert bench.parse(["--warmup", "0"]).warmup == 3
    assert bench.maybe_spawn([], 1) is None
