"""GPU parity of the time-chunked parallel scan (§6(a), Fig. 4).

Plan invariance: the same inputs under chunk lengths L = 1 (every edge a leaf:
exactly the paper's Fig. 4 tree), 2, 3, 7, 64 and E (serial) all match the fp64 oracle
within the BASELINE gates; the tree has exactly ceil(log2 P) up-sweep levels,
checked through the launch count of the logZ-only call.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset_plan():
    yield
    tsb.set_plan_chunk(0)


def run(pot_np, lengths_np, dev, L):
    tsb.set_plan_chunk(L)
    pot = torch.from_numpy(np.ascontiguousarray(pot_np)).to(dev)
    lengths = (torch.from_numpy(lengths_np.astype(np.int32)).to(dev)
               if lengths_np is not None else None)
    lz_only, fl_only = tsb.logpartition(pot, lengths)
    n_logz = tsb.last_launch_count()
    marg, lz, fl = tsb.marginals(pot, lengths)
    torch.cuda.synchronize()
    return (lz_only.cpu().numpy(), fl_only.cpu().numpy(), marg.cpu().numpy(), lz.cpu().numpy(),
            fl.cpu().numpy(), n_logz)


def check_plan(pot_np, lengths_np, dev, Ls):
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, lengths_np, threads=8)
    E = pot_np.shape[1]
    for L in Ls:
        lz_only, fl_only, marg, lz, fl, n_logz = run(pot_np, lengths_np, dev, L)
        check_logz(lz_only, lz_ref)
        check_logz(lz, lz_ref)
        assert (fl_only.astype(np.uint32) == fl_ref).all(), (L, fl_only, fl_ref)
        assert (fl.astype(np.uint32) == fl_ref).all(), (L, fl, fl_ref)
        check_marg(marg, mg_ref)
        if 0 < L < E:
            P = -(-E // L)
            H = math.ceil(math.log2(P)) if P > 1 else 0
            # memset-free launch accounting: fast summary + exact summary + H levels + root logZ
            assert n_logz == 2 + H + 1, (L, P, H, n_logz)


@pytest.mark.parametrize("B,N,C", [(32, 25, 20), (3, 200, 64), (2, 150, 128), (2, 70, 3),
                                   (2, 90, 37), (2, 300, 20), (1, 2, 5)])
def test_plan_invariance(dev, B, N, C):
    pot = tsgen.potentials(B, N, C, seed=900 + N + C)
    E = N - 1
    Ls = sorted({1, 2, 3, 7, 64, E})
    check_plan(pot, None, dev, [L for L in Ls if L <= max(E, 1)])


def test_plan_invariance_lengths_masks_flags(dev):
    B, N, C = 7, 60, 20
    pot = tsgen.tagging_potentials(B, N, C, seed=5, mask_frac=0.25)
    lengths = tsgen.random_lengths(B, N, 3)
    lengths[0], lengths[1] = 1, N
    pot[2] = -np.inf          # EMPTY
    pot[3, 10, 2, 3] = np.nan  # NONFINITE
    lengths[4] = 0             # BADLEN
    check_plan(pot, lengths, dev, [1, 3, 16, N - 1])


@pytest.mark.parametrize("C", [3, 20, 64])
def test_scan_exact_fallback_and_offsets(dev, C):
    # peaked tiles flag chunks for the exact log-space summary; 1e4 + N(0,1) needs re-centring
    check_plan(tsgen.peaked_potentials(2, 50, C, seed=C), None, dev, [1, 4, 13])
    check_plan(tsgen.large_offset_potentials(2, 50, C, seed=C), None, dev, [1, 5])


def test_cfg3_shape_chunked(dev):
    cfg = tsgen.CONFIGS[3]
    pot = tsgen.potentials(4, cfg.N, cfg.C, cfg.seed, cfg.quantum)
    check_plan(pot, None, dev, [32, 128])


def test_cfg5_shape_auto_plan_sampled(dev):
    """cfg5 geometry (B=4, C=128) on a shortened chain: the auto plan chunks it (B < #SMs)."""
    B, N, C = 4, 4097, 128
    pot = tsgen.potentials(B, N, C, seed=tsgen.CONFIGS[5].seed, s=tsgen.quantum(N - 1))
    tsb.set_plan_chunk(0)
    t = torch.from_numpy(pot).to(dev)
    marg, lz, fl = tsb.marginals(t)
    assert tsb.last_launch_count() > 2  # chunked: summaries + tree + leaf sweeps
    lz_ref, mg_ref, _ = oracle.chain_marginals(pot, threads=4)
    check_logz(lz.cpu().numpy(), lz_ref)
    check_marg(marg.cpu().numpy(), mg_ref)


@pytest.mark.parametrize("mode", [3, 1, 0])
@pytest.mark.parametrize("B,N,C", [(2, 300, 128), (3, 200, 100), (2, 97, 66)])
def test_tensor_core_summaries(dev, mode, B, N, C):
    """Leaf summaries on tcgen05 (3 = 3xTF32, 1 = 1xTF32) vs the SIMT fp32 kernel (0): all
    within the BASELINE gates of the fp64 oracle, chunked plans with ragged last chunks."""
    tsb.set_tc_summary(mode)
    try:
        pot = tsgen.potentials(B, N, C, seed=70 + C + mode)
        check_plan(pot, None, dev, [1, 7, 64])
        pot = tsgen.tagging_potentials(B, N, C, seed=3, mask_frac=0.2)
        lengths = tsgen.random_lengths(B, N, 11)
        lengths[0] = N
        check_plan(pot, lengths, dev, [5, 33])
    finally:
        tsb.set_tc_summary(3)


@pytest.mark.parametrize("mode", [3, 1])
def test_tensor_core_summaries_gate(dev, mode):
    """Peaked tiles (entries ~ -90 nats) trip the precision gate; the exact kernel redoes them."""
    tsb.set_tc_summary(mode)
    try:
        check_plan(tsgen.peaked_potentials(2, 60, 128, seed=9), None, dev, [4, 13])
        check_plan(tsgen.large_offset_potentials(2, 60, 128, seed=2), None, dev, [6])
        check_plan(20.0 * tsgen.potentials(2, 60, 128, seed=4), None, dev, [8])
    finally:
        tsb.set_tc_summary(3)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_auto_plan_per_rank_cfg3_keeps_meet64(dev, G):
    """Batch sharding of cfg3 over G ranks (B = 256 / G per rank, N = 512, C = 64): the auto
    plan keeps the one-read-per-sweep meet-in-the-middle kernel on every per-rank batch (the
    chunked SIMT scan measured 4.7x slower at B = 128; abi.cu auto_chunk)."""
    cfg = tsgen.CONFIGS[3]
    tsb.set_plan_chunk(0)
    pot = torch.empty((cfg.B // G, cfg.E, cfg.C, cfg.C), dtype=torch.float32, device=dev)
    tsgen.fill_torch(pot, cfg)
    tsb.marginals(pot)
    assert tsb.last_kernel() == "meet64_kernel"


@pytest.mark.parametrize("jump", [8.0, 30.0, 120.0])
def test_tensor_core_predicted_shift(dev, jump):
    """The tensor-core summaries shift each tile by the previous tile's max (a prediction):
    tiles whose level jumps by +-jump nats from one edge to the next (30: within the 2^40
    tolerance, no gate; 120: the prediction gate sends the chunk to the exact kernel), whole
    -inf tiles (at a chunk start and inside), and a chunk whose first tile is masked except one
    entry — all within the BASELINE gates of the fp64 oracle."""
    B, N, C = 3, 160, 128
    pot = tsgen.potentials(B, N, C, seed=int(jump))
    lvl = np.where(np.arange(N - 1) % 2 == 0, 0.0, jump).astype(np.float32)
    pot = (pot + lvl[None, :, None, None]).astype(np.float32)
    pot[1, 40] = -np.inf                    # a whole masked tile inside a chunk
    pot[2, 0] = -np.inf                     # the first tile of the first chunk ...
    pot[2, 0, 3, 5] = 1.0                   # ... except one entry
    check_plan(pot, None, dev, [40, 17])
