"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host-side path.

The partitioning, the all-gather of segment summaries and the combine order of
paper_2002_00876_b200.dist run for real across 2 processes; the per-segment compute is
injected with fp64 oracle ops (test infrastructure), so the result must equal the
unsharded oracle to fp64 rounding.  The CUDA ops behind the same interface are covered
by tests/test_segments_gpu.py (virtual segments on one GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import tsgen
from paper_2002_00876_b200 import dist as tdist


class OracleSegmentOps:
    """fp64 reference implementation of the segment summary / combine (tests only)."""

    def summary(self, local_pot, edge_begin, n_global):
        pot = local_pot.numpy()
        self.pot = pot
        return torch.from_numpy(np.stack([oracle.chain_summary(pot[b]) for b in range(pot.shape[0])]))

    def finish(self, gathered, rank, world, want_marg):
        S = gathered.numpy()  # [world, B, C, C]
        B, C = S.shape[1], S.shape[2]
        logz = np.empty(B)
        margs = []
        for b in range(B):
            a = np.zeros(C)
            for g in range(world):
                if g == rank:
                    a_in = a.copy()
                a = oracle.semiring_matmul(a[None, :], S[g, b])[0]
            m = a.max()
            logz[b] = m + np.log(np.exp(a - m).sum())
            beta = np.zeros(C)
            for g in range(world - 1, rank, -1):
                beta = oracle.semiring_matmul(S[g, b], beta[:, None])[:, 0]
            if want_marg:
                pot = self.pot[b].astype(np.float64)
                E = pot.shape[0]
                al = [a_in]
                for t in range(E):
                    al.append(oracle.semiring_matmul(al[-1][None, :], pot[t])[0])
                be = [None] * (E + 1)
                be[E] = beta
                for t in range(E - 1, -1, -1):
                    be[t] = oracle.semiring_matmul(pot[t], be[t + 1][:, None])[:, 0]
                mu = np.stack([np.exp(al[t][:, None] + pot[t] + be[t + 1][None, :] - logz[b])
                               for t in range(E)])
                margs.append(mu)
        marg = torch.from_numpy(np.stack(margs)) if want_marg else None
        return marg, torch.from_numpy(logz), torch.zeros(B, dtype=torch.int32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, N, C, seed, result_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        pot = tsgen.potentials(B, N, C, seed)
        E = N - 1
        begin, count = tdist.shard_edges(E, world, rank)
        local = torch.from_numpy(np.ascontiguousarray(pot[:, begin:begin + count]))
        marg, logz, flags = tdist.time_sharded_marginals(local, begin, N, ops=OracleSegmentOps())
        lz_ref, mg_ref, _ = oracle.chain_marginals(pot)
        ok_lz = np.allclose(logz.numpy(), lz_ref, rtol=1e-12, atol=1e-12)
        ok_mg = np.allclose(marg.numpy(), mg_ref[:, begin:begin + count], atol=1e-12)
        # logZ identical on every rank (same combine order everywhere)
        allz = [torch.zeros(B, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allz, logz.to(torch.float64))
        same = all(torch.equal(allz[0], z) for z in allz)
        # batch sharding: contiguous slices, no collective, covers the batch exactly once
        b0, b1 = tdist.shard_batch(B, world, rank)
        lzb, _, _ = oracle.chain_marginals(pot[b0:b1], want_marg=False)
        ok_b = np.allclose(lzb, lz_ref[b0:b1], rtol=1e-15)
        with open(os.path.join(result_dir, f"r{rank}"), "w") as f:
            f.write(f"{int(ok_lz)} {int(ok_mg)} {int(same)} {int(ok_b)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,N,C", [(3, 17, 4), (2, 40, 6)])
def test_time_sharded_gloo_world2(tmp_path, B, N, C):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), B, N, C, 11, str(tmp_path)), nprocs=world,
             join=True)
    for r in range(world):
        assert open(tmp_path / f"r{r}").read() == "1 1 1 1", r


def test_shard_ranges_partition():
    for n in (0, 1, 7, 64, 65535):
        for world in (1, 2, 3, 8):
            spans = [tdist.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (b0, c0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + c0 == b1
            assert sum(c for _, c in spans) == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


class OracleViterbiSegmentOps:
    """fp64 reference of the Viterbi segment steps (max-plus summary, boundary vector, local
    forward with first-index backpointers, end-label maps, local backtrack) — tests only."""

    def summary(self, local_pot, edge_begin, n_global):
        pot = local_pot.numpy()
        self.pot = pot.astype(np.float64)
        return torch.from_numpy(np.stack([oracle.chain_summary(pot[b], oracle.MAX)
                                          for b in range(pot.shape[0])]))

    def maps(self, gathered, rank, world):
        S = gathered.numpy()
        B, C = S.shape[1], S.shape[2]
        self.bp, self.zE = [], []
        maps = np.empty((B, C), np.int32)
        score = np.empty(B)
        for b in range(B):
            v = np.zeros(C)
            for g in range(world):
                if g == rank:
                    d = v.copy()
                v = np.max(v[:, None] + S[g, b], axis=0)
            score[b] = v.max()
            self.zE.append(int(np.argmax(v)))           # first argmax (reading R5)
            bps = []
            for t in range(self.pot.shape[1]):
                x = d[:, None] + self.pot[b, t]
                bps.append(np.argmax(x, axis=0))        # smallest index on ties
                d = np.max(x, axis=0)
            self.bp.append(bps)
            for j in range(C):
                z = j
                for t in range(len(bps) - 1, -1, -1):
                    z = int(bps[t][z])
                maps[b, j] = z
        return torch.from_numpy(maps), torch.from_numpy(score), torch.zeros(B, dtype=torch.int32)

    def finish(self, gathered_maps, rank, world):
        M = gathered_maps.numpy()
        B = M.shape[1]
        E = self.pot.shape[1]
        path = np.empty((B, E + 1), np.int32)
        for b in range(B):
            e = self.zE[b]
            for g in range(world - 1, rank, -1):
                e = int(M[g, b, e])
            path[b, E] = e
            for t in range(E - 1, -1, -1):
                e = int(self.bp[b][t][e])
                path[b, t] = e
        return torch.from_numpy(path)


def _vworker(rank, world, port, B, N, C, seed, result_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        pot = (np.random.default_rng(seed).integers(-3, 4, size=(B, N - 1, C, C)) * 0.5
               ).astype(np.float32)  # coarse: frequent exact ties
        begin, count = tdist.shard_edges(N - 1, world, rank)
        local = torch.from_numpy(np.ascontiguousarray(pot[:, begin:begin + count]))
        path, score, flags = tdist.time_sharded_viterbi(local, begin, N,
                                                        ops=OracleViterbiSegmentOps())
        p_ref, s_ref, _ = oracle.chain_viterbi(pot)
        ok_p = np.array_equal(path.numpy(), p_ref[:, begin:begin + count + 1])
        ok_s = np.array_equal(score.numpy(), s_ref)
        with open(os.path.join(result_dir, f"v{rank}"), "w") as f:
            f.write(f"{int(ok_p)} {int(ok_s)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,N,C", [(3, 17, 4), (2, 41, 5)])
def test_time_sharded_viterbi_gloo_world2(tmp_path, B, N, C):
    world = 2
    mp.spawn(_vworker, args=(world, _free_port(), B, N, C, 5, str(tmp_path)), nprocs=world,
             join=True)
    for r in range(world):
        assert open(tmp_path / f"v{r}").read() == "1 1", r


def _bworker(rank, world, port, B, N, C, seed, result_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        pot = tsgen.potentials(B, N, C, seed)
        b0, b1 = tdist.shard_batch(B, world, rank)

        def fn(p):  # per-rank compute (fp64 oracle: test infrastructure)
            lz, mg, fl = oracle.chain_marginals(p.numpy())
            return torch.from_numpy(mg), torch.from_numpy(lz), torch.from_numpy(fl.astype(np.int32))

        mg, lz, fl = tdist.batch_sharded(fn, torch.from_numpy(np.ascontiguousarray(pot[b0:b1])),
                                         B_global=B)
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot)
        ok = (np.array_equal(lz.numpy(), lz_ref) and np.array_equal(mg.numpy(), mg_ref)
              and np.array_equal(fl.numpy(), fl_ref.astype(np.int32)))
        with open(os.path.join(result_dir, f"b{rank}"), "w") as f:
            f.write(f"{int(ok)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [5, 2])
def test_batch_sharded_gather_gloo_world2(tmp_path, B):
    """Uneven batch shards (B = 5 over 2 ranks; B = 2) gathered back into the global batch,
    bit-identical to the unsharded computation."""
    world = 2
    mp.spawn(_bworker, args=(world, _free_port(), B, 9, 3, 21, str(tmp_path)), nprocs=world,
             join=True)
    for r in range(world):
        assert open(tmp_path / f"b{r}").read() == "1", r
