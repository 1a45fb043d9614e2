"""GPU parity of the semi-Markov CRF (Table 1 'Semi-Markov' P:44; reading
R17) through the C ABI against the fp64 oracle (oracle.semimarkov_marginals, pinned by
enumeration of segmentations x labelings): logZ 1e-5 relative, marginals 1e-4 absolute,
flags identical; K = 1 equals the linear-chain path."""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_logz, check_marg

pytestmark = pytest.mark.gpu


def _pot(B, N, K, C, seed):
    rng = np.random.default_rng(seed)
    return (rng.integers(-128, 129, size=(B, N - 1, K, C, C)) / 64.0).astype(np.float32)


def _parity(pot, dev, lengths=None):
    lz_ref, mg_ref, fl_ref = oracle.semimarkov_marginals(pot, lengths)
    lt = torch.from_numpy(lengths).to(dev) if lengths is not None else None
    mg, lz, fl = tsb.semimarkov(torch.from_numpy(pot).to(dev), lt)
    check_logz(lz.cpu().numpy(), lz_ref)
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all(), (fl.cpu().numpy(), fl_ref)
    return check_marg(mg.cpu().numpy(), mg_ref)


@pytest.mark.parametrize("B,N,K,C", [(2, 6, 3, 4), (3, 25, 4, 20), (2, 40, 8, 16),
                                     (2, 20, 16, 8), (2, 12, 3, 100), (2, 2, 4, 5),
                                     (1, 1, 2, 3), (2, 33, 5, 128), (2, 9, 3, 200)])
def test_semimarkov_parity(dev, B, N, K, C):
    err = _parity(_pot(B, N, K, C, N * K + C), dev)
    assert err < 1e-5


def test_semimarkov_k1_equals_linear_chain(dev):
    pot = tsgen.potentials(4, 25, 20, seed=5)
    mg, lz, _ = tsb.semimarkov(torch.from_numpy(np.ascontiguousarray(pot[:, :, None])).to(dev))
    m2, l2, _ = tsb.marginals(torch.from_numpy(pot).to(dev))
    assert float((lz.double() - l2.double()).abs().max()) <= 1e-5 * float(l2.abs().max())
    assert float((mg[:, :, 0] - m2).abs().max()) <= 1e-5


def test_semimarkov_lengths_flags(dev):
    B, N, K, C = 6, 15, 4, 6
    pot = _pot(B, N, K, C, 3)
    pot[2] = -np.inf                      # EMPTY
    pot[3, 5, 1, 2, 2] = np.nan           # NONFINITE (used part)
    lengths = np.array([15, 1, 15, 15, 0, 7], np.int32)
    _parity(pot, dev, lengths)


def test_semimarkov_masked_and_large_offsets(dev):
    pot = _pot(3, 20, 4, 10, 9)
    mask = np.random.default_rng(1).random(pot.shape) < 0.3
    pot[mask] = -np.inf
    _parity(pot, dev)
    _parity((pot + np.float32(1e3)).astype(np.float32), dev)


def _vit_parity(pot, dev, lengths=None):
    seg_ref, sc_ref, fl_ref = oracle.semimarkov_viterbi(pot, lengths)
    lt = torch.from_numpy(lengths).to(dev) if lengths is not None else None
    seg, sc, fl = tsb.semimarkov_viterbi(torch.from_numpy(pot).to(dev), lt)
    assert (fl.cpu().numpy().astype(np.uint32) == fl_ref).all(), (fl.cpu().numpy(), fl_ref)
    np.testing.assert_array_equal(seg.cpu().numpy(), seg_ref)
    sc = sc.cpu().numpy()
    ok = np.isnan(sc_ref)
    assert np.isnan(sc[ok]).all()
    # dyadic inputs (2^-6 grid, |partial sums| << 2^18): fp32 adds are exact -> bit-exact
    np.testing.assert_array_equal(sc[~ok], sc_ref[~ok].astype(np.float32))


@pytest.mark.parametrize("B,N,K,C", [(2, 6, 3, 4), (3, 25, 4, 20), (2, 40, 8, 16),
                                     (2, 20, 16, 8), (2, 12, 3, 100), (2, 2, 4, 5),
                                     (1, 1, 2, 3), (2, 33, 5, 128), (2, 9, 3, 200),
                                     (2, 30, 2, 256)])
def test_semimarkov_viterbi_parity(dev, B, N, K, C):
    """Semi-Markov Viterbi (R18) bit-exact against the oracle (pinned by enumeration)."""
    _vit_parity(_pot(B, N, K, C, 7 * N + K + C), dev)


def test_semimarkov_viterbi_ties_lengths_flags(dev):
    rng = np.random.default_rng(11)
    B, N, K, C = 8, 30, 4, 6
    pot = (rng.integers(-2, 3, size=(B, N - 1, K, C, C)) / 2.0).astype(np.float32)  # many ties
    lengths = rng.integers(1, N + 1, size=B).astype(np.int32)
    lengths[0], lengths[1] = 1, N
    pot[2] = -np.inf
    lengths[2] = N
    pot[3, 5, 1, 2, 3] = np.nan
    lengths[3] = N
    lengths[4] = 0
    pot[5, :, :, :, 0] = -np.inf             # label 0 unreachable after node 0
    _vit_parity(pot, dev, lengths)


def test_semimarkov_viterbi_k1_equals_chain_viterbi(dev):
    pot = tsgen.potentials(5, 40, 20, seed=9)
    seg, sc, fl = tsb.semimarkov_viterbi(torch.from_numpy(pot[:, :, None].copy()).to(dev))
    path, score, fl2 = tsb.viterbi(torch.from_numpy(pot).to(dev))
    assert torch.equal(seg, path) and torch.equal(sc, score)
