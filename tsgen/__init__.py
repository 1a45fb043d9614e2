"""tsgen — seeded synthetic inputs shared by the oracle side and the GPU side.

This module holds NO arithmetic of the method (no semiring, no log-sum-exp, no
max-plus).  It only produces potentials ell[B, N-1, C, C] (fp32) and lengths,
with the shapes of the paper's workloads (Table 1 caption, P:54:
"batch 32, N = 25, C = 20") and of BASELINE.json's configs, following the
recipe of SURVEY.md §8(d) (restated in DESIGN.md §3 and tsgen/tsgen.h).

Three bit-identical implementations of the same counter-based generator:
  * numpy (this file)             — small cases, tests
  * host C   (tsgen_host.c)       — bit-equality check, oracle on-the-fly mode
  * device CUDA (tsgen_device.cu) — bench and full-size GPU parity runs
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
SEED_BASE = 0x200200876

_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (the `configs` list, in order, 1-based)."""

    no: int
    B: int
    N: int
    C: int
    op: str  # "marg" (logZ + marginals) or "viterbi"
    label: str

    @property
    def E(self) -> int:
        return self.N - 1

    @property
    def seed(self) -> int:
        return SEED_BASE + self.no

    @property
    def quantum(self) -> int:
        return quantum(self.E)

    @property
    def tokens(self) -> int:
        return self.B * self.N


CONFIGS = {
    1: Config(1, 1, 5, 3, "marg", "linear-chain CRF batch 1, N=5, C=3, log semiring"),
    2: Config(2, 32, 25, 20, "marg", "linear-chain CRF batch 32, N=25, C=20 logZ + marginals"),
    3: Config(3, 256, 512, 64, "marg", "linear-chain CRF batch 256, N=512, C=64 logZ + marginals"),
    4: Config(4, 64, 1024, 256, "viterbi", "Viterbi max-plus batch 64, N=1024, C=256"),
    5: Config(5, 4, 65536, 128, "marg", "long-sequence CRF batch 4, N=65536, C=128"),
}


def quantum(E: int) -> int:
    """Largest s in [0, 15] with E * 4 * 2^s <= 2^24 (tsgen.h: tsgen_quantum)."""
    E = max(int(E), 1)
    s = 15
    while s > 0 and E * 4 * (1 << s) > (1 << 24):
        s -= 1
    return s


def _splitmix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def values_at(seed: int, s: int, idx: np.ndarray) -> np.ndarray:
    """Dyadic fp32 values for an array of global uint64 indices."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = _splitmix64(np.uint64(seed) + (idx + np.uint64(1)) * GOLDEN)
    m = np.uint64(0xFFFF)
    k = ((x & m).astype(np.int64) + ((x >> np.uint64(16)) & m).astype(np.int64)
         + ((x >> np.uint64(32)) & m).astype(np.int64) + (x >> np.uint64(48)).astype(np.int64)
         - 131070)
    k = k >> (15 - s)  # arithmetic shift on int64 == floor division by 2^(15-s)
    return (k.astype(np.float32) * np.float32(1.0 / (1 << s))).astype(np.float32)


def potentials(B: int, N: int, C: int, seed: int, s: int | None = None, t_begin: int = 0,
               E_local: int | None = None, E_global: int | None = None) -> np.ndarray:
    """ell[B, E_local, C, C] fp32 (numpy), global edge indices t_begin..t_begin+E_local-1."""
    E = N - 1
    if E_global is None:
        E_global = E
    if E_local is None:
        E_local = E_global - t_begin
    if s is None:
        s = quantum(E_global)
    b = np.arange(B, dtype=np.uint64)[:, None, None, None]
    t = (np.arange(E_local, dtype=np.uint64) + np.uint64(t_begin))[None, :, None, None]
    i = np.arange(C, dtype=np.uint64)[None, None, :, None]
    j = np.arange(C, dtype=np.uint64)[None, None, None, :]
    CC = np.uint64(C)
    idx = ((b * np.uint64(E_global) + t) * CC + i) * CC + j
    return values_at(seed, s, idx)


def config_potentials(cfg: Config) -> np.ndarray:
    return potentials(cfg.B, cfg.N, cfg.C, cfg.seed, cfg.quantum)


# --------------------------------------------------------------------------------------
# Correctness-only input variants (SURVEY.md §8(d) "Correctness-only extras").
# Seeded numpy Generators; dyadic where Viterbi bit-exactness is asserted.
# --------------------------------------------------------------------------------------

def random_lengths(B: int, N: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(1, N + 1, size=B).astype(np.int32)


def tagging_potentials(B: int, N: int, C: int, seed: int, mask_frac: float = 0.1,
                       s: int = 6) -> np.ndarray:
    """ell[b,t,i,j] = u[b,t+1,j] + W[i,j] with ~mask_frac of W at -inf (never a full row/col).

    Emission + transition structure of a tagger (the paper's sequence-labelling use,
    P:57), values on a 2^-s grid so partial sums stay exact.
    """
    rng = np.random.default_rng(seed)
    E = N - 1
    u = rng.integers(-2 << s, (2 << s) + 1, size=(B, N, C)).astype(np.float32) / np.float32(1 << s)
    W = rng.integers(-2 << s, (2 << s) + 1, size=(C, C)).astype(np.float32) / np.float32(1 << s)
    if C > 1:
        mask = rng.random((C, C)) < mask_frac
        for r in range(C):  # never a full row or column
            if mask[r].all():
                mask[r, rng.integers(C)] = False
        for c in range(C):
            if mask[:, c].all():
                mask[rng.integers(C), c] = False
        W = np.where(mask, np.float32(-np.inf), W).astype(np.float32)
    ell = u[:, 1:, None, :] + W[None, None, :, :]
    assert ell.shape == (B, E, C, C)
    return np.ascontiguousarray(ell.astype(np.float32))


def large_offset_potentials(B: int, N: int, C: int, seed: int, offset: float = 1e4) -> np.ndarray:
    """ell = offset + N(0,1) in fp32 (catches a missing per-tile re-centring)."""
    rng = np.random.default_rng(seed)
    return (np.float32(offset) + rng.standard_normal((B, N - 1, C, C)).astype(np.float32)).astype(
        np.float32)


def wide_potentials(B: int, N: int, C: int, seed: int, scale: float = 200.0) -> np.ndarray:
    """ell = scale * N(0,1): within-tile spreads of hundreds of nats (underflow gates)."""
    rng = np.random.default_rng(seed)
    return (np.float32(scale) * rng.standard_normal((B, N - 1, C, C)).astype(np.float32)).astype(
        np.float32)


def peaked_potentials(B: int, N: int, C: int, seed: int, p_keep: float = 0.15,
                      drop: float = 90.0) -> np.ndarray:
    """Mostly-suppressed tiles: ~p_keep of the entries near 0, the rest near -drop.

    Linear-space partial sums of the dominant-label paths then fall below 2^-60 whenever
    a column's surviving entries sit on rows the running vector has suppressed, which
    exercises the exact per-cell-max recomputation (the underflow gate)
    while every non-negligible marginal stays well conditioned in fp32.
    """
    rng = np.random.default_rng(seed)
    keep = rng.random((B, N - 1, C, C)) < p_keep
    hi = rng.uniform(-1.0, 1.0, size=keep.shape)
    lo = -drop - rng.uniform(0.0, 10.0, size=keep.shape)
    return np.where(keep, hi, lo).astype(np.float32)


# --------------------------------------------------------------------------------------
# Native fills (host C and device CUDA), for bit-equality tests and full-size inputs.
# --------------------------------------------------------------------------------------

_host_lib = None
_dev_lib = None


def _load(name: str):
    path = os.path.join(_HERE, name)
    if not os.path.exists(path):
        raise RuntimeError(f"tsgen: {path} not built (run __graft_entry__.build())")
    return ctypes.CDLL(path)


def host_lib():
    global _host_lib
    if _host_lib is None:
        lib = _load("libtsgen_host.so")
        lib.tsgen_fill_host.restype = ctypes.c_int
        lib.tsgen_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.c_int64, ctypes.c_int64]
        lib.tsgen_quantum_c.restype = ctypes.c_int
        lib.tsgen_quantum_c.argtypes = [ctypes.c_int64]
        _host_lib = lib
    return _host_lib


def dev_lib():
    global _dev_lib
    if _dev_lib is None:
        lib = _load("libtsgen_device.so")
        lib.tsgen_fill_device.restype = ctypes.c_int
        lib.tsgen_fill_device.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        _dev_lib = lib
    return _dev_lib


def fill_host(B: int, N: int, C: int, seed: int, s: int | None = None, t_begin: int = 0,
              E_local: int | None = None, E_global: int | None = None) -> np.ndarray:
    E = N - 1
    E_global = E if E_global is None else E_global
    E_local = (E_global - t_begin) if E_local is None else E_local
    s = quantum(E_global) if s is None else s
    out = np.empty((B, E_local, C, C), dtype=np.float32)
    rc = host_lib().tsgen_fill_host(out.ctypes.data, B, E_local, C, seed, s, t_begin, E_global)
    if rc != 0:
        raise ValueError(f"tsgen_fill_host failed ({rc})")
    return out


def fill_device(out_ptr: int, B: int, E_local: int, C: int, seed: int, s: int, t_begin: int,
                E_global: int, stream: int = 0) -> None:
    """Fill a device buffer (raw pointer) on `stream` (raw cudaStream_t handle)."""
    rc = dev_lib().tsgen_fill_device(ctypes.c_void_p(out_ptr), B, E_local, C, seed, s, t_begin,
                                     E_global, ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"tsgen_fill_device failed ({rc})")


def fill_torch(t, cfg_or_seed, s: int | None = None, t_begin: int = 0, E_global: int | None = None):
    """Fill a contiguous torch tensor [B, E_local, C, C] (cuda) with generator values."""
    import torch  # plumbing only

    assert t.is_cuda and t.is_contiguous() and t.dtype == torch.float32 and t.dim() == 4
    B, E_local, C, _ = t.shape
    seed = cfg_or_seed.seed if isinstance(cfg_or_seed, Config) else int(cfg_or_seed)
    if E_global is None:
        E_global = t_begin + E_local
    if s is None:
        s = quantum(E_global)
    fill_device(t.data_ptr(), B, E_local, C, seed, s, t_begin, E_global,
                torch.cuda.current_stream(t.device).cuda_stream)
    return t


def fill_torch_batch(t, cfg: Config, b_begin: int):
    """Fill sequences [b_begin, b_begin + t.shape[0]) of a config's batch (global indices:
    the rank's slice of a batch-sharded input equals that slice of the unsharded one).  The
    flat index ((b·E + t)·C + i)·C + j is contiguous in b, so the slice is one [1, nb·E]
    'chain' starting at edge b_begin·E of a B·E-edge index space (same values, same s)."""
    nb, E, C, _ = t.shape
    assert E == cfg.E and C == cfg.C and 0 <= b_begin and b_begin + nb <= cfg.B
    fill_torch(t.view(1, nb * E, C, C), cfg.seed, cfg.quantum, t_begin=b_begin * E,
               E_global=cfg.B * E)
    return t
