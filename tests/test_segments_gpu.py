"""GPU: the time-sharded path with "virtual segments" on one GPU.

G segments of one chain run ts_segment_summary independently; their summaries are
concatenated on the device (standing in for the NCCL all_gather_into_tensor of
paper_2002_00876_b200.dist); each segment then runs ts_segment_finish.  Together they must
reproduce the unsharded oracle (logZ identical on every segment; marginals per segment).
This exercises every line of the time-sharded path except the collective itself.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg
from paper_2002_00876_b200 import dist as tdist

pytestmark = pytest.mark.gpu


def virtual_segments(pot_np, G, dev, want_marg=True):
    B, E, C, _ = pot_np.shape
    N = E + 1
    segs = []
    for r in range(G):
        begin, count = tdist.shard_edges(E, G, r)
        local = torch.from_numpy(np.ascontiguousarray(pot_np[:, begin:begin + count])).to(dev)
        segs.append((begin, count, tsb.Segment(local, begin, N)))
    summaries = torch.stack([s.summary() for (_, _, s) in segs])  # "all_gather"
    outs = [s.finish(summaries, r, G, want_marg) for r, (_, _, s) in enumerate(segs)]
    torch.cuda.synchronize()
    return segs, outs


@pytest.mark.parametrize("B,N,C,G", [(4, 257, 64, 2), (2, 1001, 128, 8), (3, 120, 20, 4),
                                     (2, 50, 3, 8), (2, 9, 37, 8),
                                     # B*C*C odd: the fp64 offsets follow a padded matrix
                                     # section (was a misaligned-address fault)
                                     (1, 40, 5, 2), (1, 60, 37, 4), (3, 31, 5, 3)])
def test_virtual_segments_match_unsharded(dev, B, N, C, G):
    pot = tsgen.potentials(B, N, C, seed=31 + G)
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot, threads=8)
    segs, outs = virtual_segments(pot, G, dev)
    lz0 = outs[0][1].cpu().numpy()
    for (begin, count, _), (marg, logz, flags) in zip(segs, outs):
        lz = logz.cpu().numpy()
        assert (lz == lz0).all()  # bit-identical across segments
        check_logz(lz, lz_ref)
        assert (flags.cpu().numpy() == 0).all()
        check_marg(marg.cpu().numpy(), mg_ref[:, begin:begin + count])


def test_virtual_segments_chunked_and_logz_only(dev):
    B, N, C, G = 2, 700, 64, 2
    pot = tsgen.potentials(B, N, C, seed=5)
    lz_ref, mg_ref, _ = oracle.chain_marginals(pot, threads=8)
    try:
        tsb.set_plan_chunk(23)  # several chunks (and a tree) inside every segment
        segs, outs = virtual_segments(pot, G, dev)
        for (begin, count, _), (marg, logz, _) in zip(segs, outs):
            check_logz(logz.cpu().numpy(), lz_ref)
            check_marg(marg.cpu().numpy(), mg_ref[:, begin:begin + count])
        _, outs = virtual_segments(pot, G, dev, want_marg=False)
        for (_, logz, _) in outs:
            check_logz(logz.cpu().numpy(), lz_ref)
    finally:
        tsb.set_plan_chunk(0)


def test_virtual_segments_flags(dev):
    B, N, C, G = 3, 90, 20, 3
    pot = tsgen.potentials(B, N, C, seed=8)
    pot[1] = -np.inf          # EMPTY everywhere
    pot[2, 70, 3, 4] = np.nan  # NONFINITE in the last segment only
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot)
    segs, outs = virtual_segments(pot, G, dev)
    for (begin, count, _), (marg, logz, flags) in zip(segs, outs):
        check_logz(logz.cpu().numpy(), lz_ref)
        assert (flags.cpu().numpy().astype(np.uint32) == fl_ref).all()
        check_marg(marg.cpu().numpy(), mg_ref[:, begin:begin + count])


def test_cfg5_generated_segments_sampled(dev):
    """cfg5 geometry: B=4, C=128, per-rank slices generated in place by global edge index
    (tsgen), shortened to N=8193 so the fp64 oracle finishes in seconds."""
    cfg = tsgen.CONFIGS[5]
    B, N, C, G = cfg.B, 8193, cfg.C, 8
    E = N - 1
    s = tsgen.quantum(E)
    segs = []
    for r in range(G):
        begin, count = tdist.shard_edges(E, G, r)
        local = torch.empty((B, count, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(local, cfg.seed, s, t_begin=begin, E_global=E)
        segs.append((begin, count, tsb.Segment(local, begin, N)))
    summ = torch.stack([sg.summary() for (_, _, sg) in segs])
    outs = [sg.finish(summ, r, G) for r, (_, _, sg) in enumerate(segs)]
    torch.cuda.synchronize()
    for b in (0, 3):
        edges = [1, segs[3][0], segs[3][0] + 7, E - 1]
        lz_ref, ed, m_ref, _ = oracle.gen_marginals(cfg.seed, s, b, N, C, edges)
        for (begin, count, _), (marg, logz, _) in zip(segs, outs):
            check_logz(logz[b:b + 1].cpu().numpy(), [lz_ref])
            for e_i, e in enumerate(ed):
                if begin <= e < begin + count:
                    check_marg(marg[b, e - begin].cpu().numpy(), m_ref[e_i])


# ---------------------------------------------------------------- time-sharded Viterbi

def virtual_viterbi(pot_np, G, dev):
    """The time-sharded Viterbi flow (dist.time_sharded_viterbi) with the two all-gathers
    replaced by device-side stacks; returns the stitched global path, scores, flags."""
    B, E, C, _ = pot_np.shape
    N = E + 1
    segs = []
    for r in range(G):
        begin, count = tdist.shard_edges(E, G, r)
        local = torch.from_numpy(np.ascontiguousarray(pot_np[:, begin:begin + count])).to(dev)
        segs.append((begin, count, tsb.ViterbiSegment(local, begin, N)))
    summ = torch.stack([s.summary() for (_, _, s) in segs])            # all_gather 1
    res = [s.maps(summ, r, G) for r, (_, _, s) in enumerate(segs)]
    maps = torch.stack([m for (m, _, _) in res])                        # all_gather 2
    paths = [s.finish(maps, r, G) for r, (_, _, s) in enumerate(segs)]
    torch.cuda.synchronize()
    full = np.full((B, N), -2, np.int32)
    for (begin, count, _), p in zip(segs, paths):
        p = p.cpu().numpy()
        seg_part = full[:, begin:begin + count + 1]
        overlap = seg_part != -2
        assert (seg_part[overlap] == p[overlap]).all()  # shared boundary nodes agree
        full[:, begin:begin + count + 1] = p
    scores = [sc.cpu().numpy() for (_, sc, _) in res]
    flags = [fl.cpu().numpy() for (_, _, fl) in res]
    return full, scores, flags


@pytest.mark.parametrize("B,N,C,G", [(3, 257, 64, 2), (2, 1001, 128, 8), (3, 120, 20, 4),
                                     (2, 50, 3, 8), (2, 9, 37, 8), (4, 64, 5, 3)])
def test_virtual_viterbi_segments_bit_exact(dev, B, N, C, G):
    pot = tsgen.potentials(B, N, C, seed=71 + G)
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot, threads=8)
    full, scores, flags = virtual_viterbi(pot, G, dev)
    np.testing.assert_array_equal(full, p_ref)
    for sc, fl in zip(scores, flags):
        assert (sc == s_ref.astype(np.float32)).all()  # identical on every segment
        assert (fl.astype(np.uint32) == f_ref).all()
    # and equal to the unsharded GPU path
    path, score, _ = tsb.viterbi(torch.from_numpy(pot).to(dev))
    np.testing.assert_array_equal(path.cpu().numpy(), full)


def test_virtual_viterbi_ties_and_flags(dev):
    # coarse dyadic values: many exact ties (reading R5, smallest index wins)
    B, N, C, G = 4, 80, 6, 4
    pot = (np.random.default_rng(3).integers(-2, 3, size=(B, N - 1, C, C)) * 0.5).astype(np.float32)
    pot[1] = -np.inf                                  # EMPTY
    pot[2, 40, 1, 2] = np.nan                         # NONFINITE (in the 3rd segment)
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot, threads=4)
    full, scores, flags = virtual_viterbi(pot, G, dev)
    for b in (0, 3):
        np.testing.assert_array_equal(full[b], p_ref[b])
        assert scores[0][b] == np.float32(s_ref[b])
    assert (full[1] == -1).all() and (full[2] == -1).all()
    for fl in flags:
        assert (fl.astype(np.uint32) == f_ref).all()
