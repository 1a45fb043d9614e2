"""GPU: cfg5 at FULL size (B=4, N=65536, C=128; BASELINE.json configs[4]) — logZ and
marginals against the fp64 oracle in generator mode (pinned in test_oracle_gen_pins.py).

BJ asks for tolerance-matched logZ and marginals "on every config"; the long-chain plan is
the time-chunked scan of §6(a): P = ceil(#SMs / B) chunks whose 3xTF32
tensor-core summaries feed the Fig. 4 tree.  Its rounding accumulates over
1772-edge chunks and a 6-level tree, so this checks the real plan, not a shortened one:

  * logZ of all 4 sequences (|ΔA| <= 1e-5·max(1,|A|), reading R7);
  * μ element-wise (1e-4 abs, R8) on 4 edges inside EVERY chunk — its first two, a
    middle one and its last — so both sides of every chunk boundary are compared;
  * Σ_ij μ_t = 1 on every one of the 4 × 65535 edges;
  * the same for the 8-way time-sharded flow with virtual segments at
    full N: each segment's own chunked plan, summaries stacked in place of the NCCL
    all-gather, logZ bit-identical on all segments.
"""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg
from paper_2002_00876_b200 import dist as tdist

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CFG = tsgen.CONFIGS[5]
G = 8


def plan_chunks(E, B, sms):
    """The default plan's chunking (abi.cu log_plan): P = ceil(sms/B), L = ceil(E/P)."""
    P = min(-(-sms // B), -(-E // 32))
    L = -(-E // P)
    return [(k * L, min((k + 1) * L, E)) for k in range(-(-E // L))]


def probe_edges(ranges):
    out = set()
    for lo, hi in ranges:
        out.update(e for e in (lo, lo + 1, (lo + hi) // 2, hi - 1) if lo <= e < hi)
    return out


@pytest.fixture(scope="module")
def reference(dev):
    E = CFG.E
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    chunks = plan_chunks(E, CFG.B, sms)
    edges = probe_edges(chunks)
    for r in range(G):  # segment boundaries and each segment's own chunk boundaries
        begin, count = tdist.shard_edges(E, G, r)
        edges |= {begin + lo for lo, hi in plan_chunks(count, CFG.B, sms)}
        edges |= {begin + hi - 1 for lo, hi in plan_chunks(count, CFG.B, sms)}
        edges |= {begin, begin + count - 1}
    edges = sorted(edges)

    def one(b):
        return oracle.gen_marginals(CFG.seed, CFG.quantum, b, CFG.N, CFG.C, edges)

    with cf.ThreadPoolExecutor(CFG.B) as ex:
        res = list(ex.map(one, range(CFG.B)))
    assert all(f == 0 for (_, _, _, f) in res)
    return chunks, np.asarray(edges), res


def check_sampled(marg_b, lz_b, ref_b, edge_offset=0, count=None):
    lz_ref, ed, m_ref, _ = ref_b
    check_logz([lz_b], [lz_ref])
    n = 0
    for k, e in enumerate(ed):
        el = int(e) - edge_offset
        if 0 <= el < (count if count is not None else marg_b.shape[0]):
            check_marg(marg_b[el].cpu().numpy(), m_ref[k])
            n += 1
    return n


def test_cfg5_full_default_plan(dev, reference):
    chunks, edges, ref = reference
    assert len(chunks) >= 8  # the real multi-chunk plan (37 chunks at 148 SMs)
    pot = torch.empty((CFG.B, CFG.E, CFG.C, CFG.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, CFG)
    marg, logz, flags = tsb.marginals(pot)
    torch.cuda.synchronize()
    del pot
    assert (flags.cpu().numpy() == 0).all()
    sums = marg.sum(dim=(2, 3), dtype=torch.float64)
    assert float((sums - 1).abs().max()) < 1e-4
    lz = logz.cpu().numpy()
    for b in range(CFG.B):
        n = check_sampled(marg[b], float(lz[b]), ref[b])
        assert n == len(edges)
    del marg
    torch.cuda.empty_cache()


def test_cfg5_full_virtual_segments(dev, reference):
    _, edges, ref = reference
    E, N, C, B = CFG.E, CFG.N, CFG.C, CFG.B
    segs = []
    for r in range(G):
        begin, count = tdist.shard_edges(E, G, r)
        local = torch.empty((B, count, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(local, CFG.seed, CFG.quantum, t_begin=begin, E_global=E)
        segs.append((begin, count, tsb.Segment(local, begin, N)))
    summ = torch.stack([sg.summary() for (_, _, sg) in segs])  # stands in for all_gather
    lz0 = None
    covered = 0
    for r, (begin, count, sg) in enumerate(segs):
        marg, logz, flags = sg.finish(summ, r, G)
        torch.cuda.synchronize()
        assert (flags.cpu().numpy() == 0).all()
        lz = logz.cpu().numpy()
        if lz0 is None:
            lz0 = lz
        assert (lz == lz0).all()  # bit-identical on every segment
        sums = marg.sum(dim=(2, 3), dtype=torch.float64)
        assert float((sums - 1).abs().max()) < 1e-4
        for b in range(B):
            covered += check_sampled(marg[b], float(lz[b]), ref[b], begin, count)
        del marg
        sg.pot = None
    assert covered == B * len(edges)
    torch.cuda.empty_cache()
