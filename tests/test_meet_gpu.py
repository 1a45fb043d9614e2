"""GPU parity of the meet-in-the-middle marginals kernel (fb_meet.cu, C = 64, one serial
chunk per sequence) against the fp64 oracle, and against the two-kernel sweep path.

The serial plan is forced with the chunk knob (L >= N-1), so small batches take the same
kernel as BASELINE cfg3 (B=256, where the automatic plan is already serial).  Cases cover
the midpoint split at every parity of E_b (E_b = 0, 1, 2, 3, ...), ragged lengths, flags,
masks, the shift re-verification path (tile maxima jumping by > 28 nats between steps), the
underflow gate and the product-form fallbacks of the marginal epilogue.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg

pytestmark = pytest.mark.gpu

C = 64


@pytest.fixture
def serial_plan():
    tsb.set_plan_chunk(1 << 40)
    tsb.set_meet(True)
    yield
    tsb.set_plan_chunk(0)
    tsb.set_meet(True)


def run(pot_np, lengths_np, dev, meet=True):
    tsb.set_meet(meet)
    pot = torch.from_numpy(np.ascontiguousarray(pot_np)).to(dev)
    lengths = (torch.from_numpy(lengths_np.astype(np.int32)).to(dev)
               if lengths_np is not None else None)
    m, lz, fl = tsb.marginals(pot, lengths)
    n = tsb.last_launch_count()
    return m.cpu().numpy(), lz.cpu().numpy(), fl.cpu().numpy().astype(np.uint32), n


def check(pot_np, lengths_np, dev):
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot_np, lengths_np, threads=8)
    m, lz, fl, n = run(pot_np, lengths_np, dev, meet=True)
    assert n == 1, "meet kernel must be a single launch"
    check_logz(lz, lz_ref)
    assert (fl == fl_ref).all(), (fl, fl_ref)
    err = check_marg(m, mg_ref)
    # the two-kernel sweep path agrees within the same gates
    m2, lz2, fl2, n2 = run(pot_np, lengths_np, dev, meet=False)
    assert n2 >= 2
    check_logz(lz2, lz_ref)
    assert (fl2 == fl_ref).all()
    check_marg(m2, mg_ref)
    return err


@pytest.mark.parametrize("N", [2, 3, 4, 5, 6, 17, 64, 130, 513])
def test_meet_shapes(dev, serial_plan, N):
    pot = tsgen.potentials(3, N, C, seed=700 + N)
    check(pot, None, dev)


def test_meet_lengths_every_midpoint_parity(dev, serial_plan):
    B, N = 12, 40
    pot = tsgen.potentials(B, N, C, seed=41)
    lengths = np.array([1, 2, 3, 4, 5, 6, 7, 20, 21, 39, 40, 33], dtype=np.int32)
    check(pot, lengths, dev)


def test_meet_flags(dev, serial_plan):
    B, N = 7, 30
    pot = tsgen.potentials(B, N, C, seed=9)
    pot[1] = -np.inf                     # EMPTY
    pot[2, 3, 1, 2] = np.nan             # NONFINITE, early edge (forward phase-1 half)
    pot[3, N - 3, 0, 0] = np.inf         # +inf late edge (backward phase-1 half)
    pot[6, 20, 5, 7] = np.nan            # NaN in the backward half
    lengths = np.full(B, N, dtype=np.int32)
    lengths[4] = 0                       # BADLEN
    lengths[5] = N + 1                   # BADLEN
    check(pot, lengths, dev)


def test_meet_masked(dev, serial_plan):
    pot = tsgen.tagging_potentials(4, 50, C, seed=64, mask_frac=0.3)
    check(pot, tsgen.random_lengths(4, 50, 3), dev)


def test_meet_large_offset_and_shift(dev, serial_plan):
    check(tsgen.large_offset_potentials(3, 60, C, seed=C), None, dev)
    base = tsgen.potentials(3, 50, C, seed=31, s=6)
    for c in (1e4, -1e4):
        check((base + np.float32(c)).astype(np.float32), None, dev)


def test_meet_shift_jumps_redo_path(dev, serial_plan):
    # per-edge offsets jumping by 0 / +45 / -60 nats: the lagged shift fails its check
    # (|T - T_s| log2 e > 40) on many steps of both engines and the step is redone
    B, N = 3, 48
    pot = tsgen.potentials(B, N, C, seed=5).astype(np.float64)
    off = np.array([0.0, 45.0, -15.0, 30.0, -30.0, 2.0])[np.arange(N - 1) % 6]
    pot += off[None, :, None, None]
    check(pot.astype(np.float32), None, dev)


def test_meet_peaked_gate(dev, serial_plan):
    check(tsgen.peaked_potentials(3, 40, C, seed=C), None, dev)


def test_meet_wide(dev, serial_plan):
    check(tsgen.wide_potentials(2, 40, C, seed=C, scale=20.0), None, dev)


def test_meet_cfg3_reduced(dev, serial_plan):
    cfg = tsgen.CONFIGS[3]
    pot = tsgen.potentials(5, cfg.N, cfg.C, cfg.seed, cfg.quantum)
    check(pot, None, dev)


def test_meet_deterministic(dev, serial_plan):
    pot = torch.from_numpy(tsgen.potentials(4, 200, C, seed=3)).to(dev)
    a = tsb.marginals(pot)
    b = tsb.marginals(pot)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
