"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by
element on seeded inputs.  Every test here needs a B200.

Sizes: oracle-complete at sizes spanning several tiles and a ragged tail; full
BASELINE.json sizes on sampled sequences / property checks.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg, check_viterbi

pytestmark = pytest.mark.gpu


def to_dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def run_all(pot_np, lengths_np, dev, marg=True):
    pot = to_dev(pot_np, dev)
    lengths = to_dev(lengths_np.astype(np.int32), dev) if lengths_np is not None else None
    out = {}
    if marg:
        m, lz, fl = tsb.marginals(pot, lengths)
        out["marg"], out["logz"], out["flags"] = m.cpu().numpy(), lz.cpu().numpy(), fl.cpu().numpy()
    lz2, fl2 = tsb.logpartition(pot, lengths)
    out["logz_only"], out["flags_only"] = lz2.cpu().numpy(), fl2.cpu().numpy()
    return out


def assert_log_parity(pot_np, lengths_np, dev, marg=True):
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, lengths_np, want_marg=marg, threads=8)
    out = run_all(pot_np, lengths_np, dev, marg)
    check_logz(out["logz_only"], lz_ref)
    assert (out["flags_only"].astype(np.uint32) == fl_ref).all(), (out["flags_only"], fl_ref)
    if marg:
        check_logz(out["logz"], lz_ref)
        assert (out["flags"].astype(np.uint32) == fl_ref).all()
        return check_marg(out["marg"], mg_ref)


def assert_viterbi_parity(pot_np, lengths_np, dev):
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot_np, lengths_np, threads=8)
    pot = to_dev(pot_np, dev)
    lengths = to_dev(lengths_np.astype(np.int32), dev) if lengths_np is not None else None
    path, score, flags = tsb.viterbi(pot, lengths)
    check_viterbi(path.cpu().numpy(), score.cpu().numpy(), p_ref, s_ref)
    assert (flags.cpu().numpy().astype(np.uint32) == f_ref).all()
    # max-semiring entry points: logZ = score, marginals = one-hot indicator of the path
    lz, _ = tsb.logpartition(pot, lengths, semiring="max")
    check_viterbi(path.cpu().numpy(), lz.cpu().numpy(), p_ref, s_ref)
    m, lz2, _ = tsb.marginals(pot, lengths, semiring="max")
    np.testing.assert_array_equal(m.cpu().numpy(),
                                  oracle.max_indicator(p_ref, pot_np.shape[-1], lengths_np))


# ------------------------------------------------------------------ BASELINE configs

def test_generator_device_equals_numpy(dev):
    for (B, N, C, seed, s) in [(2, 7, 5, 123, 15), (3, 40, 20, 9, 13), (1, 9, 64, 4, 12)]:
        t = torch.empty((B, N - 1, C, C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(t, seed, s)
        assert t.cpu().numpy().tobytes() == tsgen.potentials(B, N, C, seed, s).tobytes()


def test_cfg1_brute_scale(dev):
    cfg = tsgen.CONFIGS[1]
    pot = tsgen.config_potentials(cfg)
    err = assert_log_parity(pot, None, dev)
    assert err < 1e-5
    assert_viterbi_parity(pot, None, dev)


def test_cfg2_full(dev):
    cfg = tsgen.CONFIGS[2]
    pot = tsgen.config_potentials(cfg)
    assert_log_parity(pot, None, dev)
    assert_viterbi_parity(pot, None, dev)


@pytest.mark.parametrize("B,N,C", [(3, 130, 64), (2, 77, 20), (2, 41, 128), (4, 33, 3),
                                   (2, 600, 20), (3, 17, 37), (2, 9, 1), (2, 50, 100)])
def test_streaming_and_small_shapes(dev, B, N, C):
    pot = tsgen.potentials(B, N, C, seed=5000 + N + C)
    assert_log_parity(pot, None, dev)
    assert_viterbi_parity(pot, None, dev)


def test_cfg3_reduced_elementwise(dev):
    cfg = tsgen.CONFIGS[3]
    pot = tsgen.potentials(6, cfg.N, cfg.C, cfg.seed, cfg.quantum)
    assert_log_parity(pot, None, dev)
    assert_viterbi_parity(pot, None, dev)


@pytest.mark.parametrize("B,N,C", [(2, 70, 130), (3, 40, 200), (2, 30, 256), (2, 2, 256)])
def test_log_semiring_wide_labels(dev, B, N, C):
    """128 < C <= 256 on chains that do not fit one CTA: fb_wide (forward / backward recursion
    CTAs with the exact per-cell LSE, then a machine-wide marginal pass)."""
    pot = tsgen.potentials(B, N, C, seed=900 + N + C)
    assert_log_parity(pot, None, dev)
    lengths = np.array([N] + [max(1, N // 3)] * (B - 1), np.int32)
    assert_log_parity(pot, lengths, dev)
    pot[0, N // 2 - 1, 3, 4] = np.nan
    assert_log_parity(pot, None, dev)


@pytest.mark.parametrize("C", [131, 256])
def test_log_wide_labels_masks_flags_ranges(dev, C):
    """fb_wide (128 < C <= 256): masks, EMPTY / NONFINITE / BADLEN / len-1 rows, offsets,
    peaked and wide-range inputs; C = 131 takes the scalar (C*C % 4 != 0) marginal path."""
    B, N = 7, 45
    pot = tsgen.tagging_potentials(B, N, C, seed=C, mask_frac=0.2)
    lengths = tsgen.random_lengths(B, N, C)
    lengths[0], lengths[1] = 1, N
    pot[2] = -np.inf
    lengths[2] = N
    pot[3, 7, 2, 1] = np.inf
    lengths[3] = N
    lengths[4] = 0
    lengths[5] = N + 2
    assert_log_parity(pot, lengths, dev)
    assert_log_parity(tsgen.large_offset_potentials(2, 30, C, seed=C), None, dev)
    assert_log_parity(tsgen.peaked_potentials(2, 30, C, seed=C), None, dev)
    assert_log_parity(tsgen.wide_potentials(2, 30, C, seed=C, scale=50.0), None, dev)


@pytest.mark.parametrize("C", [132, 200, 256])
def test_log_wide_ring_matches_register_path(dev, C):
    """The two wide-label sweeps (SMEM ring / registers) both match the oracle."""
    pot = tsgen.potentials(3, 50, C, seed=31 + C)
    lengths = np.array([50, 17, 1], np.int32)
    try:
        for ring in (True, False):
            tsb.set_wide_ring(ring)
            assert_log_parity(pot, lengths, dev)
    finally:
        tsb.set_wide_ring(True)


def test_log_wide_cfg4_shape_full(dev):
    """logZ + marginals at cfg4's full shape (B64 N1024 C256, the log semiring) through
    fb_wide; oracle on sampled sequences (first, last) element by element, every sequence's
    marginals sum to 1 per edge."""
    cfg = tsgen.CONFIGS[4]
    pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, cfg)
    m, lz, fl = tsb.marginals(pot)
    assert tsb.last_kernel() == "fb_wide_sweep_kernel"
    assert (fl.cpu().numpy() == 0).all()
    sums = m.sum(dim=(2, 3), dtype=torch.float64)
    assert float((sums - 1).abs().max()) < 1e-4
    lz = lz.cpu().numpy()
    CC = cfg.C * cfg.C
    for b in (0, cfg.B - 1):
        idx = np.arange(b * cfg.E * CC, (b + 1) * cfg.E * CC, dtype=np.uint64)
        pb = tsgen.values_at(cfg.seed, cfg.quantum, idx).reshape(1, cfg.E, cfg.C, cfg.C)
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pb, None, threads=8)
        check_logz(lz[b:b + 1], lz_ref)
        check_marg(m[b:b + 1].cpu().numpy(), mg_ref)
    del pot, m
    torch.cuda.empty_cache()


@pytest.mark.parametrize("C", [3, 20, 64, 130, 256])
def test_viterbi_shapes(dev, C):
    pot = tsgen.potentials(3, 70, C, seed=77 + C)
    assert_viterbi_parity(pot, None, dev)


def test_cfg4_viterbi_full(dev):
    cfg = tsgen.CONFIGS[4]
    pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, cfg)
    path, score, flags = tsb.viterbi(pot)
    path, score = path.cpu().numpy(), score.cpu().numpy()
    del pot
    torch.cuda.empty_cache()
    assert (flags.cpu().numpy() == 0).all()
    import concurrent.futures as cf

    def one(b):
        return oracle.gen_viterbi(cfg.seed, cfg.quantum, b, cfg.N, cfg.C)

    with cf.ThreadPoolExecutor(8) as ex:
        res = list(ex.map(one, range(cfg.B)))
    for b, (p, s, f) in enumerate(res):
        assert f == 0
        np.testing.assert_array_equal(path[b], p)
        assert score[b] == np.float32(s)


def test_viterbi_full_size_cfg2_cfg3_cfg5(dev):
    """Bit-exact Viterbi on every BASELINE config (BJ: "bit-exact Viterbi ... on every
    config"): cfg2 and cfg3 complete, cfg5 (B=4, N=65536, C=128) complete, oracle in
    generator mode (no 17 GB host buffer)."""
    import concurrent.futures as cf

    for no in (2, 3, 5):
        cfg = tsgen.CONFIGS[no]
        pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
        tsgen.fill_torch(pot, cfg)
        path, score, flags = tsb.viterbi(pot)
        path, score = path.cpu().numpy(), score.cpu().numpy()
        del pot
        torch.cuda.empty_cache()
        assert (flags.cpu().numpy() == 0).all()
        bs = range(cfg.B) if no != 3 else (0, 1, 137, 254, 255)

        def one(b, cfg=cfg):
            return oracle.gen_viterbi(cfg.seed, cfg.quantum, b, cfg.N, cfg.C)

        with cf.ThreadPoolExecutor(8) as ex:
            res = list(ex.map(one, bs))
        for b, (p, s, f) in zip(bs, res):
            assert f == 0
            np.testing.assert_array_equal(path[b], p)
            assert score[b] == np.float32(s)


def test_cfg3_full_sampled(dev):
    cfg = tsgen.CONFIGS[3]
    pot = torch.empty((cfg.B, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, cfg)
    marg, logz, flags = tsb.marginals(pot)
    assert (flags.cpu().numpy() == 0).all()
    sums = marg.sum(dim=(2, 3))
    assert float((sums - 1).abs().max()) < 1e-4  # every edge sums to 1
    logz = logz.cpu().numpy()
    for b in (0, 137, 255):
        lz_ref, edges, m_ref, f = oracle.gen_marginals(cfg.seed, cfg.quantum, b, cfg.N, cfg.C,
                                                       range(cfg.E))
        check_logz(logz[b:b + 1], [lz_ref])
        check_marg(marg[b].cpu().numpy(), m_ref)


# ------------------------------------------------------------------ edge cases

def test_variable_lengths(dev):
    for (B, N, C, seed) in [(8, 25, 20, 1), (6, 90, 64, 2), (5, 40, 128, 3), (7, 300, 8, 4)]:
        pot = tsgen.potentials(B, N, C, seed=seed)
        lengths = tsgen.random_lengths(B, N, seed)
        lengths[0] = 1
        lengths[1] = N
        assert_log_parity(pot, lengths, dev)
        assert_viterbi_parity(pot, lengths, dev)


def test_flags_empty_nonfinite_badlen(dev):
    for (N, C) in [(25, 20), (70, 64), (8, 3)]:
        B = 6
        pot = tsgen.potentials(B, N, C, seed=9)
        pot[1] = -np.inf                           # EMPTY
        pot[2, N // 2, 1 % C, 2 % C] = np.nan      # NONFINITE
        pot[3, 1, 0, 0] = np.inf                   # +inf -> NONFINITE
        lengths = np.full(B, N, dtype=np.int32)
        lengths[4] = 0                             # BADLEN
        lengths[5] = N + 1                         # BADLEN
        assert_log_parity(pot, lengths, dev)
        assert_viterbi_parity(pot, lengths, dev)


def test_masked_tagging_inputs(dev):
    for (B, N, C) in [(4, 25, 20), (3, 100, 64), (2, 20, 7)]:
        pot = tsgen.tagging_potentials(B, N, C, seed=C, mask_frac=0.3)
        assert_log_parity(pot, None, dev)
        assert_viterbi_parity(pot, None, dev)


@pytest.mark.parametrize("C", [3, 20, 64])
def test_large_offset_recentring(dev, C):
    # l = 1e4 + N(0,1): fails the 1e-4 marginal gate without per-tile re-centring (§7.3-7)
    pot = tsgen.large_offset_potentials(3, 60, C, seed=C)
    assert_log_parity(pot, None, dev)


@pytest.mark.parametrize("C", [3, 20, 64, 128])
def test_peaked_inputs_exercise_underflow_gate(dev, C):
    pot = tsgen.peaked_potentials(3, 40, C, seed=C)
    assert_log_parity(pot, None, dev)


@pytest.mark.parametrize("C", [3, 20, 64, 128])
def test_wide_inputs(dev, C):
    # within-tile spreads of ~100 nats: |ah|, |bh| reach ~2^7, fp32 storage costs
    # ~ulp(128) per term in the marginal exponent (precision envelope)
    pot = tsgen.wide_potentials(2, 40, C, seed=C, scale=20.0)
    assert_log_parity(pot, None, dev)


def test_shift_by_1e4(dev):
    # magnitude 1e4 -> finite results equal to the shifted result + analytic shift
    for C in (20, 64):
        base = tsgen.potentials(3, 50, C, seed=31, s=6)
        for c in (1e4, -1e4):
            assert_log_parity((base + np.float32(c)).astype(np.float32), None, dev)


def test_deterministic_bitwise(dev):
    for (B, N, C) in [(32, 25, 20), (4, 200, 64)]:
        pot = to_dev(tsgen.potentials(B, N, C, seed=3), dev)
        a = tsb.marginals(pot)
        b = tsb.marginals(pot)
        for x, y in zip(a, b):
            assert torch.equal(x, y)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("shape", [(32, 25, 20), (6, 200, 64), (3, 9, 5)])
def test_host_buffers_end_to_end(dev, shape, graphs):
    """ts_marginals_host: chunked pipeline, eager on the 1st sighting of a binding, captured
    on the 2nd, graph replay after; fresh input contents in the same pinned buffers must be
    read on every call (nothing cached but the launch sequence)."""
    B, N, C = shape
    pot = torch.empty((B, N - 1, C, C), dtype=torch.float32).pin_memory()
    marg = torch.empty_like(pot).pin_memory()
    logz = torch.empty(B, dtype=torch.float32).pin_memory()
    flags = torch.empty(B, dtype=torch.int32).pin_memory()
    lengths = torch.empty(B, dtype=torch.int32).pin_memory()
    tsb.set_host_graphs(graphs)
    try:
        for call in range(4):
            pot_np = tsgen.potentials(B, N, C, seed=100 + call)
            len_np = tsgen.random_lengths(B, N, 7 + call)
            pot.copy_(torch.from_numpy(pot_np))
            lengths.copy_(torch.from_numpy(len_np))
            tsb.marginals_host(pot, marg, logz, flags, lengths_host=lengths if call % 2 else None,
                               device=dev)
            torch.cuda.synchronize()
            lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, len_np if call % 2 else None)
            check_logz(logz.numpy(), lz_ref)
            check_marg(marg.numpy(), mg_ref)
            np.testing.assert_array_equal(flags.numpy(), fl_ref)
    finally:
        tsb.set_host_graphs(True)


@pytest.mark.parametrize("pipeline", [2, 1, 0])
def test_host_pipeline_back_to_back(dev, pipeline):
    """Cross-call copy pipeline of ts_marginals_host (single-chunk payloads): 6 calls
    enqueued back to back WITHOUT synchronising, alternating between two input/output
    buffer sets and rewriting host inputs only after the call that read them completed,
    with and without graph replay; every result matches the oracle."""
    B, N, C = 32, 25, 20
    sets = []
    for _ in range(3):
        sets.append(tuple(torch.empty(sh, dtype=dt).pin_memory() for sh, dt in
                          [((B, N - 1, C, C), torch.float32), ((B, N - 1, C, C), torch.float32),
                           ((B,), torch.float32), ((B,), torch.int32)]))
    refs = {}
    tsb.set_host_pipeline(pipeline)
    try:
        for graphs in (True, False):
            tsb.set_host_graphs(graphs)
            events = []
            for call in range(6):
                pot, marg, logz, flags = sets[call % 3]
                if call >= 3:
                    events[call - 3].synchronize()   # the call that read this input is done
                    k = call - 3
                    lz_ref, mg_ref, fl_ref = refs[k]
                    p_, m_, l_, f_ = sets[k % 3]
                    check_logz(l_.numpy(), lz_ref)
                    check_marg(m_.numpy(), mg_ref)
                    np.testing.assert_array_equal(f_.numpy(), fl_ref)
                pot_np = tsgen.potentials(B, N, C, seed=500 + call + 10 * graphs)
                pot.copy_(torch.from_numpy(pot_np))
                refs[call] = oracle.chain_marginals(pot_np)
                tsb.marginals_host(pot, marg, logz, flags, device=dev)
                ev = torch.cuda.Event()
                ev.record()
                events.append(ev)
            torch.cuda.synchronize()
            for k in range(3, 6):
                lz_ref, mg_ref, fl_ref = refs[k]
                p_, m_, l_, f_ = sets[k % 3]
                check_logz(l_.numpy(), lz_ref)
                check_marg(m_.numpy(), mg_ref)
    finally:
        tsb.set_host_graphs(True)
        tsb.set_host_pipeline(True)


def test_host_pipeline_binding_changes(dev):
    """Pipelined host calls interleaved with calls of other shapes (a different workspace
    layout) on the same workspace, enqueued without synchronising: every result is right."""
    shapes = [(32, 25, 20), (5, 40, 12), (32, 25, 20), (64, 300, 20), (32, 25, 20)]
    ws = tsb.Workspace(dev)
    outs = []
    for k, (B, N, C) in enumerate(shapes):
        pot_np = tsgen.potentials(B, N, C, seed=900 + k)
        pot = torch.from_numpy(pot_np).pin_memory()
        marg = torch.empty_like(pot).pin_memory()
        logz = torch.empty(B, dtype=torch.float32).pin_memory()
        flags = torch.empty(B, dtype=torch.int32).pin_memory()
        tsb.marginals_host(pot, marg, logz, flags, device=dev, ws=ws)
        outs.append((pot_np, marg, logz, flags))
    torch.cuda.synchronize()
    for pot_np, marg, logz, flags in outs:
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, None, threads=8)
        check_logz(logz.numpy(), lz_ref)
        check_marg(marg.numpy(), mg_ref)
        np.testing.assert_array_equal(flags.numpy(), fl_ref)


@pytest.mark.parametrize("G", [2, 4])
def test_cluster_dsmem_variant(dev, G):
    """The chunked-scan plan for short chains on a G-CTA cluster (fb_cscan.cu: chunk
    summaries exchanged by DSMEM bulk copies); shapes it cannot chunk run one CTA."""
    try:
        tsb.set_small_cluster(G)
        for (B, N, C) in [(32, 25, 20), (3, 40, 7), (2, 17, 32)]:
            assert_log_parity(tsgen.potentials(B, N, C, seed=G + C), None, dev)
        pot = tsgen.tagging_potentials(6, 30, 12, seed=4, mask_frac=0.3)
        lengths = tsgen.random_lengths(6, 30, 9)
        pot[1] = -np.inf
        pot[2, 5, 1, 1] = np.nan
        lengths[3] = 1
        lengths[4] = 0
        assert_log_parity(pot, lengths, dev)
        assert_log_parity(tsgen.peaked_potentials(2, 30, 20, seed=1), None, dev)
        assert_log_parity(tsgen.large_offset_potentials(2, 30, 20, seed=2), None, dev)
    finally:
        tsb.set_small_cluster(0)


def test_host_calls_switching_streams(dev):
    """ts_marginals_host calls alternating between two torch streams without synchronising
    (same hidden workspace and device staging): each call orders after the previous one on
    the other stream, so every result is right."""
    B, N, C = 32, 25, 20
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = []
    for k in range(8):
        pot_np = tsgen.potentials(B, N, C, seed=1300 + k)
        pot = torch.from_numpy(pot_np).pin_memory()
        marg = torch.empty_like(pot).pin_memory()
        logz = torch.empty(B, dtype=torch.float32).pin_memory()
        flags = torch.empty(B, dtype=torch.int32).pin_memory()
        with torch.cuda.stream(streams[k % 2]):
            tsb.marginals_host(pot, marg, logz, flags, device=dev)
        outs.append((pot_np, marg, logz, flags))
    torch.cuda.synchronize()
    for pot_np, marg, logz, flags in outs:
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np)
        check_logz(logz.numpy(), lz_ref)
        check_marg(marg.numpy(), mg_ref)
        np.testing.assert_array_equal(flags.numpy(), fl_ref)


def test_host_graph_key_covers_kernel_knobs(dev):
    """A repeated host binding replays its graph, but toggling a kernel-selection knob
    (ts_set_tiny) must re-enqueue with the newly selected kernel, not replay the old one."""
    B, N, C = 32, 25, 20
    pot_np = tsgen.potentials(B, N, C, seed=1400)
    pot = torch.from_numpy(pot_np).pin_memory()
    marg = torch.empty_like(pot).pin_memory()
    logz = torch.empty(B, dtype=torch.float32).pin_memory()
    flags = torch.empty(B, dtype=torch.int32).pin_memory()
    lz_ref, mg_ref, _ = oracle.chain_marginals(pot_np)
    try:
        tsb.set_host_pipeline(False)
        for _ in range(3):  # eager, capture, replay
            tsb.marginals_host(pot, marg, logz, flags, device=dev)
        torch.cuda.synchronize()
        k_tiny = tsb.last_kernel()
        tsb.set_tiny(0)
        tsb.marginals_host(pot, marg, logz, flags, device=dev)
        torch.cuda.synchronize()
        k_small = tsb.last_kernel()
        assert k_tiny != k_small, (k_tiny, k_small)
        check_logz(logz.numpy(), lz_ref)
        check_marg(marg.numpy(), mg_ref)
    finally:
        tsb.set_tiny(1)
        tsb.set_host_pipeline(True)


@pytest.mark.parametrize("with_flags", [True, False])
def test_host_contiguous_outputs_one_copy(dev, with_flags):
    """ts_marginals_host with the outputs back to back in one pinned block (marg | logZ |
    flags): logZ / flags are written behind the device marginals and return in the same copy;
    back-to-back calls with fresh inputs, BADLEN / EMPTY rows, against the oracle."""
    B, N, C = 32, 25, 20
    nel = B * (N - 1) * C * C
    blk = tsb.host_empty((nel + 2 * B,))
    marg = blk[:nel].view(B, N - 1, C, C)
    logz = blk[nel:nel + B]
    flags = blk[nel + B:].view(torch.int32) if with_flags else None
    pot = tsb.host_empty((B, N - 1, C, C))
    lengths = tsb.host_empty((B,), torch.int32)
    for call in range(5):
        pot_np = tsgen.potentials(B, N, C, seed=500 + call)
        pot_np[3] = -np.inf                    # EMPTY
        len_np = tsgen.random_lengths(B, N, 9 + call).astype(np.int32)
        len_np[5] = 0                          # BADLEN
        pot.copy_(torch.from_numpy(pot_np))
        lengths.copy_(torch.from_numpy(len_np))
        tsb.marginals_host(pot, marg, logz, flags, lengths_host=lengths, device=dev)
        torch.cuda.synchronize()
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, len_np)
        check_logz(logz.numpy(), lz_ref)
        check_marg(marg.numpy(), mg_ref)
        if with_flags:
            np.testing.assert_array_equal(flags.numpy().astype(np.uint32), fl_ref)


def test_host_pipeline_modes_interleaved(dev):
    """Host calls switching pipeline mode (three-stage, two-stream, stream-ordered) and
    output layout (back to back, separate) between calls, enqueued without synchronising on
    the same workspace: every result matches the oracle."""
    B, N, C = 32, 25, 20
    nel = B * (N - 1) * C * C
    calls = []
    try:
        for k, mode in enumerate([2, 2, 1, 2, 0, 2, 1, 1, 2]):
            tsb.set_host_pipeline(mode)
            pot_np = tsgen.potentials(B, N, C, seed=900 + k)
            pot = tsb.host_empty((B, N - 1, C, C))
            pot.copy_(torch.from_numpy(pot_np))
            if k % 2:
                blk = tsb.host_empty((nel + 2 * B,))
                outs = (blk[:nel].view(B, N - 1, C, C), blk[nel:nel + B], blk[nel + B:].view(torch.int32))
            else:
                outs = (tsb.host_empty((B, N - 1, C, C)), tsb.host_empty((B,)), tsb.host_empty((B,), torch.int32))
            tsb.marginals_host(pot, *outs, device=dev)
            calls.append((pot_np, pot, outs))
        torch.cuda.synchronize()
    finally:
        tsb.set_host_pipeline(True)
    for pot_np, _, (m, l, f) in calls:
        lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np)
        check_logz(l.numpy(), lz_ref)
        check_marg(m.numpy(), mg_ref)
        np.testing.assert_array_equal(f.numpy().astype(np.uint32), fl_ref)
