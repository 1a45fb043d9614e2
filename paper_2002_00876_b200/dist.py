"""Multi-GPU partitioning of the hot path: one process per GPU,
torch.distributed (NCCL over NVLink / NVSwitch) for the plumbing.

* Batch sharding: sequences are independent — each rank runs its contiguous slice of the
  batch; no data-path collective (weak scaling in bench.py).
* Time sharding (long chains, BASELINE cfg5): rank r owns a contiguous range of edges of
  every sequence.  Each rank computes its segment's C x C transfer matrix (the semiring
  product of its edges, the §6(a) scan applied across devices), ONE
  all_gather_into_tensor exchanges the summaries, and every rank combines them in the same
  order (identical logZ on all ranks) before running its local sweeps.

The compute is injected (`ops`) so the host-side partitioning / gather / combine plumbing
can be exercised on CPU with gloo in tests; the default ops are the CUDA kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of n items: (begin, count) of `rank`."""
    base, extra = divmod(int(n), int(world))
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def shard_batch(B: int, world: int, rank: int) -> tuple[int, int]:
    b0, nb = shard_range(B, world, rank)
    return b0, b0 + nb


def shard_edges(E: int, world: int, rank: int) -> tuple[int, int]:
    """Edges [begin, begin + count) of a chain with E edges owned by `rank`."""
    return shard_range(E, world, rank)


class CudaSegmentOps:
    """Default ops: the sm_100a kernels through the C ABI (ts_segment_summary/finish)."""

    def __init__(self):
        self.seg = None

    def summary(self, local_pot, edge_begin, n_global):
        from . import Segment

        self.seg = Segment(local_pot, edge_begin, n_global)
        return self.seg.summary()

    def finish(self, gathered, rank, world, want_marg):
        return self.seg.finish(gathered, rank, world, want_marg)


def _all_gather(t: torch.Tensor, group) -> torch.Tensor:
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
    try:
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    except (RuntimeError, NotImplementedError, ValueError):  # backends without the fused op
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t.contiguous(), group=group)
        out = torch.stack(parts)
    return out


def time_sharded_marginals(local_pot, edge_begin: int, n_global: int, group=None,
                           want_marg: bool = True, ops=None):
    """Marginals / logZ of chains split in time across the ranks of `group`.

    local_pot: this rank's edges [edge_begin, edge_begin + E_local) of every sequence.
    Returns (marg for the local edges or None, logz [B] (global, identical on all ranks), flags).
    """
    ops = ops or CudaSegmentOps()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    summ = ops.summary(local_pot, edge_begin, n_global)
    gathered = _all_gather(summ, group)
    return ops.finish(gathered, rank, world, want_marg)


class CudaViterbiSegmentOps:
    """Default ops for time-sharded Viterbi: ts_segment_viterbi_summary / _maps / _finish."""

    def __init__(self):
        self.seg = None

    def summary(self, local_pot, edge_begin, n_global):
        from . import ViterbiSegment

        self.seg = ViterbiSegment(local_pot, edge_begin, n_global)
        return self.seg.summary()

    def maps(self, gathered, rank, world):
        return self.seg.maps(gathered, rank, world)

    def finish(self, gathered_maps, rank, world):
        return self.seg.finish(gathered_maps, rank, world)


def time_sharded_viterbi(local_pot, edge_begin: int, n_global: int, group=None, ops=None):
    """Viterbi of chains split in time across the ranks of `group`:
    all-gather of the max-plus segment summaries, then of the [B, C] end-label maps.
    Returns (local path [B, E_local + 1] covering global nodes edge_begin..., global score
    [B], flags [B]); the score and flags are identical on every rank."""
    ops = ops or CudaViterbiSegmentOps()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    summ = ops.summary(local_pot, edge_begin, n_global)
    maps, score, flags = ops.maps(_all_gather(summ, group), rank, world)
    path = ops.finish(_all_gather(maps, group), rank, world)
    return path, score, flags


def all_gather_batch(t: torch.Tensor, B_global: int, group=None) -> torch.Tensor:
    """Concatenate every rank's batch slice (rank r holds rows shard_batch(B_global, world, r))
    into the global [B_global, ...] tensor on every rank: slices are padded to the largest
    shard, all-gathered once, and cut back in rank order."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b0, b1 = shard_batch(B_global, world, rank)
    assert t.shape[0] == b1 - b0, (t.shape, b0, b1)
    cmax = max(shard_range(B_global, world, r)[1] for r in range(world))
    pad = torch.zeros((cmax,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    g = _all_gather(pad, group)  # [world, cmax, ...]
    return torch.cat([g[r, : shard_range(B_global, world, r)[1]] for r in range(world)])


def batch_sharded(fn, pot_local, *args, B_global: int | None = None, group=None, **kw):
    """Batch sharding: sequences are independent, so each rank runs `fn` on its
    own contiguous slice (shard_batch) with no collective on the data path.  With
    `B_global` set, every tensor `fn` returns (leading dimension = the local batch) is
    all-gathered into the global batch afterwards (all_gather_batch) — an output gather,
    not part of the computation."""
    out = fn(pot_local, *args, **kw)
    if B_global is None:
        return out
    if isinstance(out, torch.Tensor):
        return all_gather_batch(out, B_global, group)
    return tuple(all_gather_batch(o, B_global, group) if isinstance(o, torch.Tensor) else o
                 for o in out)
