"""GPU parity of the latency-optimised short-chain kernels (C % 4 == 0, C <= 28) against the
fp64 oracle, and against the general single-CTA kernel (fb_small.cu) they replace on those
shapes: every test runs three times — one CTA per sequence (fb_tiny.cu) and the §6(a)
chunked scan on a 2- and a 4-CTA cluster per sequence (fb_cscan.cu; shapes it cannot chunk,
and gated / non-finite sequences, take its in-launch exact fallback).  Gates as everywhere
(DESIGN.md §5): logZ 1e-5 relative, marginals 1e-4 absolute, flags identical.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg

pytestmark = pytest.mark.gpu

TINY_C = [4, 8, 12, 16, 20, 24, 28]


@pytest.fixture(autouse=True, params=[0, 2, 4], ids=["tiny", "cscan2", "cscan4"])
def plan(request):
    tsb.set_small_cluster(request.param)
    yield request.param
    tsb.set_small_cluster(0)


@pytest.fixture
def tiny_off():
    tsb.set_tiny(False)
    yield
    tsb.set_tiny(True)


def parity(pot_np, lengths_np, dev):
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, lengths_np, threads=8)
    pot = torch.from_numpy(np.ascontiguousarray(pot_np)).to(dev)
    lengths = (torch.from_numpy(lengths_np.astype(np.int32)).to(dev)
               if lengths_np is not None else None)
    m, lz, fl = tsb.marginals(pot, lengths)
    check_logz(lz.cpu().numpy(), lz_ref)
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all(), (fl.cpu().numpy(), fl_ref)
    err = check_marg(m.cpu().numpy(), mg_ref)
    lz2, fl2 = tsb.logpartition(pot, lengths)
    check_logz(lz2.cpu().numpy(), lz_ref)
    assert (fl2.cpu().numpy().astype(np.uint32) == fl_ref).all()
    return err, m


@pytest.mark.parametrize("C", TINY_C)
@pytest.mark.parametrize("N", [1, 2, 3, 17, 25, 40])
def test_tiny_shapes(dev, C, N):
    pot = tsgen.potentials(3, N, C, seed=700 + 31 * C + N)
    err, _ = parity(pot, None, dev)
    assert err < 1e-5


@pytest.mark.parametrize("C", [4, 20, 28])
def test_tiny_lengths_and_flags(dev, C):
    B, N = 9, 30
    pot = tsgen.potentials(B, N, C, seed=C + 1)
    lengths = tsgen.random_lengths(B, N, C)
    lengths[0], lengths[1] = 1, N
    pot[2] = -np.inf                   # EMPTY
    pot[3, 4, 1, 2] = np.nan           # NONFINITE
    pot[4, 0, 0, 0] = np.inf           # NONFINITE
    lengths[5] = 0                     # BADLEN
    lengths[6] = N + 3                 # BADLEN
    lengths[2] = lengths[3] = lengths[4] = N
    parity(pot, lengths, dev)


@pytest.mark.parametrize("C", [8, 20])
def test_tiny_masked_offset_peaked_wide(dev, C):
    parity(tsgen.tagging_potentials(4, 25, C, seed=C, mask_frac=0.3), None, dev)
    parity(tsgen.large_offset_potentials(3, 25, C, seed=C), None, dev)
    parity(tsgen.peaked_potentials(3, 25, C, seed=C), None, dev)
    parity(tsgen.wide_potentials(2, 25, C, seed=C, scale=20.0), None, dev)
    base = tsgen.potentials(3, 25, C, seed=31, s=6)
    for c in (1e4, -1e4):
        parity((base + np.float32(c)).astype(np.float32), None, dev)


@pytest.mark.parametrize("C", [4, 20])
def test_tiny_hidden_path_gates(dev, C):
    """A label reachable only through a column of -200 nats followed by a row of +200:
    the linear sweep underflows there (EX = 0), so the exact log-space step (sweep gate)
    and the exact log-space edge (marginal gate) must recover the path's mass."""
    B, N = 4, 25
    pot = tsgen.potentials(B, N, C, seed=77, s=10)
    for b in range(B):
        t, j = 5 + 3 * b, (b + 1) % C
        pot[b, t, :, j] = -200.0
        pot[b, t + 1, j, :] = 200.0 + pot[b, t + 1, j, :]
    pot[3, 2, :, :] = -300.0 + pot[3, 2, :, :]      # a whole tile far below its neighbours
    parity(pot.astype(np.float32), None, dev)


def test_tiny_matches_general_kernel(dev, tiny_off):
    for C in TINY_C:
        pot = torch.from_numpy(tsgen.potentials(5, 25, C, seed=C)).to(dev)
        tsb.set_tiny(False)
        m0, l0, f0 = tsb.marginals(pot)
        tsb.set_tiny(True)
        m1, l1, f1 = tsb.marginals(pot)
        assert torch.equal(f0, f1)
        assert float((l0.double() - l1.double()).abs().max()) <= 1e-5 * float(l0.abs().max())
        assert float((m0 - m1).abs().max()) <= 2e-6


def test_tiny_cfg2_sum_to_one_and_deterministic(dev):
    cfg = tsgen.CONFIGS[2]
    pot = torch.from_numpy(tsgen.config_potentials(cfg)).to(dev)
    m, lz, fl = tsb.marginals(pot)
    s = m.double().sum(dim=(2, 3))
    assert float((s - 1).abs().max()) < 1e-5
    m2, lz2, fl2 = tsb.marginals(pot)
    assert torch.equal(m, m2) and torch.equal(lz, lz2)


def test_plan_knob_selects_kernel_for_cfg2(dev, plan):
    """cfg2 (B=32, N=25, C=20): the auto plan (-1) runs the chunked scan on 4-CTA clusters,
    the default (0) one CTA per sequence."""
    pot = torch.from_numpy(tsgen.config_potentials(tsgen.CONFIGS[2])).to(dev)
    tsb.set_small_cluster(-1)
    tsb.marginals(pot)
    assert tsb.last_kernel() == "fb_cscan_kernel"
    tsb.set_small_cluster(0)
    tsb.marginals(pot)
    assert tsb.last_kernel() == "fb_tiny_kernel"


@pytest.mark.parametrize("C", [12, 20])
def test_mixed_fast_and_fallback_sequences(dev, C):
    """One batch where some clusters take the fast chunked path and others fall back
    in-launch (a gated hidden path, a NaN, a sequence too short to chunk)."""
    B, N = 8, 33
    pot = tsgen.potentials(B, N, C, seed=90 + C, s=10)
    lengths = np.full(B, N, dtype=np.int32)
    pot[1, 9, :, 2] = -200.0
    pot[1, 10, 2, :] = 200.0 + pot[1, 10, 2, :]
    pot[3, 20, 0, 1] = np.nan
    lengths[5] = 4
    lengths[6] = 2 * 4 + 1
    parity(pot.astype(np.float32), lengths, dev)


def _chain_run(pot, steps, early, lengths=None):
    """x_{i+1} = marginals(x_i) back to back on one stream (each call reads the buffer the
    previous call is writing), plus independent calls on rotating buffers; no host sync."""
    tsb.set_tiny_early(early)
    try:
        xs = [pot]
        lzs = []
        for _ in range(steps):
            m, lz, fl = tsb.marginals(xs[-1], lengths)
            xs.append(m)
            lzs.append(lz)
        indep = [tsb.marginals(pot + float(k), lengths)[1] for k in range(8)]
        torch.cuda.synchronize()
        return xs, lzs, indep
    finally:
        tsb.set_tiny_early(True)


@pytest.mark.parametrize("C", [8, 20])
def test_tiny_early_reads_chained_calls(dev, C, plan):
    """Consecutive calls overlap (PDL) and read their inputs before waiting for the previous
    call when no recent call's outputs overlap them: a call whose potentials are the previous
    call's marginals must still see them complete — identical to waiting first, and the
    first link checked against the oracle."""
    B, N = 6, 25
    pot_np = tsgen.potentials(B, N, C, seed=41 + C)
    lengths_np = np.array([N, N - 3, 1, N, 7, N], np.int32)
    pot = torch.from_numpy(pot_np).to(dev)
    lengths = torch.from_numpy(lengths_np).to(dev)
    xs1, lz1, ind1 = _chain_run(pot, 12, True, lengths)
    xs0, lz0, ind0 = _chain_run(pot, 12, False, lengths)
    for a, b in zip(xs1, xs0):
        assert torch.equal(a, b)
    for a, b in zip(lz1 + ind1, lz0 + ind0):
        assert torch.equal(torch.nan_to_num(a, nan=7.0), torch.nan_to_num(b, nan=7.0))
    x1 = xs1[1].cpu().numpy()
    lz_ref, mg_ref, _ = oracle.chain_marginals(x1, lengths_np, threads=8)
    check_logz(lz1[1].cpu().numpy(), lz_ref)
    check_marg(xs1[2].cpu().numpy(), mg_ref)


def test_tiny_early_war_hazard(dev, plan):
    """A call whose marginal buffer is the potentials of a call that may still be running
    (write-after-read) must not write them before that call has read them; nor may it write
    the logZ buffer an earlier call is writing (write-after-write)."""
    B, N, C = 32, 25, 20
    x_np = tsgen.potentials(B, N, C, seed=77)
    y_np = tsgen.potentials(B, N, C, seed=78)
    lz_x, mg_x, _ = oracle.chain_marginals(x_np, threads=8)
    lz_y, mg_y, _ = oracle.chain_marginals(y_np, threads=8)
    for _ in range(3):
        x = torch.from_numpy(x_np).to(dev)
        y = torch.from_numpy(y_np).to(dev)
        torch.cuda.synchronize()
        m1, l1, f1 = tsb.marginals(x)           # reads x
        m2, l2, f2 = tsb.marginals(y, out=x)    # overwrites x with y's marginals
        torch.cuda.synchronize()
        check_logz(l1.cpu().numpy(), lz_x)
        check_marg(m1.cpu().numpy(), mg_x)
        check_logz(l2.cpu().numpy(), lz_y)
        check_marg(m2.cpu().numpy(), mg_y)


def test_tiny_early_graph_replay_and_streams(dev, plan):
    """Overlapping calls captured into a CUDA graph and replayed (the bench's pattern: calls on
    rotating buffers, some reading what an earlier call in the graph wrote), and calls on two
    streams joined by events: identical to the same calls made eagerly one after another."""
    B, N, C = 8, 25, 20
    pots = [torch.from_numpy(tsgen.potentials(B, N, C, seed=300 + k)).to(dev) for k in range(4)]
    outs = [torch.empty_like(pots[0]) for _ in range(6)]
    lzs = [torch.empty(B, device=dev) for _ in range(6)]

    def calls(st):
        with torch.cuda.stream(st):
            for k in range(6):
                src = pots[k % 4] if k < 4 else outs[k - 4]  # calls 4, 5 read calls 0, 1's output
                tsb.marginals(src, out=outs[k])
                lzs[k].copy_(tsb.logpartition(src)[0])

    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    calls(side)
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs], [z.clone() for z in lzs]
    for o in outs:
        o.zero_()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.graph(g, stream=cap):
        calls(torch.cuda.current_stream(dev))
    for _ in range(2):
        for o in outs:
            o.zero_()
        g.replay()
        torch.cuda.synchronize()
        for a, b in zip(outs, ref[0]):
            assert torch.equal(a, b)
        for a, b in zip(lzs, ref[1]):
            assert torch.equal(a, b)
    # two streams: the second stream's call reads the first stream's output after an event
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    s1.wait_stream(torch.cuda.current_stream(dev))
    s2.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s1):
        m1, _, _ = tsb.marginals(pots[0])
        ev = torch.cuda.Event()
        ev.record(s1)
        tsb.marginals(pots[1])  # more work behind it on s1
    with torch.cuda.stream(s2):
        s2.wait_event(ev)
        m2, _, _ = tsb.marginals(m1)
    torch.cuda.synchronize()
    assert torch.equal(m1, ref[0][0])
    assert torch.equal(m2, ref[0][4])


def _mixed_run(early, pots, feat):
    tsb.set_tiny_early(early)
    try:
        outs = []
        x = pots[0]
        for k in range(10):
            m, lz, fl = tsb.marginals(pots[k % 3])
            h = tsb.entropy(pots[(k + 1) % 3])[0]
            ex = tsb.expectation(pots[(k + 2) % 3], feat)[0]
            lz2 = tsb.logpartition(x)[0]
            x = m  # the next logpartition reads these marginals
            outs += [m, lz, fl, h, ex, lz2]
        torch.cuda.synchronize()
        return [o.clone() for o in outs]
    finally:
        tsb.set_tiny_early(True)


def test_tiny_early_mixed_entry_points(dev, plan):
    """Back-to-back marginals / entropy / expectation (fused epilogue variants) / logZ-only
    calls, some reading what an earlier call wrote, none synchronised: identical to the same
    sequence with every call waiting first."""
    B, N, C = 16, 25, 20
    pots = [torch.from_numpy(tsgen.potentials(B, N, C, seed=60 + k)).to(dev) for k in range(3)]
    feat = torch.from_numpy(tsgen.potentials(B, N, C, seed=99)).to(dev)
    a = _mixed_run(True, pots, feat)
    b = _mixed_run(False, pots, feat)
    for x, y in zip(a, b):
        assert torch.equal(torch.nan_to_num(x.float(), nan=7.0), torch.nan_to_num(y.float(), nan=7.0))
