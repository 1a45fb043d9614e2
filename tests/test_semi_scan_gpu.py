"""Semi-Markov CRF on the scan (P:44 with P:311 "Similar parallel approach
can also be used for ... semi-Markov"): the expanded-state chain (semi_expand.cu, S = C K
states) through the linear-chain plans — the chunked scan with tensor-core summaries, the
Fig. 4 tree (L = 1), the serial sweeps of the expanded chain — against the fp64 oracle
(oracle.semimarkov_marginals / semimarkov_viterbi, pinned by enumeration), plan invariance
across chunk lengths, and the segmental one-CTA kernels on the same inputs.  Gates as
everywhere: logZ 1e-5 relative, marginals 1e-4 absolute, Viterbi bit-exact (dyadic inputs).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
from _util import check_logz, check_marg

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset():
    yield
    tsb.set_plan_chunk(0)


def _pot(B, N, K, C, seed, q=64.0):
    rng = np.random.default_rng(seed)
    return (rng.integers(-128, 129, size=(B, N - 1, K, C, C)) / q).astype(np.float32)


def _marg(pot, dev, lengths, L):
    tsb.set_plan_chunk(L)
    lt = torch.from_numpy(lengths).to(dev) if lengths is not None else None
    mg, lz, fl = tsb.semimarkov(torch.from_numpy(pot).to(dev), lt)
    return mg.cpu().numpy(), lz.cpu().numpy(), fl.cpu().numpy().astype(np.uint32), tsb.last_kernel()


def test_long_chain_auto_plan_is_the_scan(dev):
    """N = 4097, K = 4, C = 20 (S = 80): the auto plan expands and chunks (tensor-core
    summaries for 64 < S <= 128); parity with the oracle."""
    B, N, K, C = 2, 4097, 4, 20
    pot = _pot(B, N, K, C, 4097, q=256.0)
    lz_ref, mg_ref, fl_ref = oracle.semimarkov_marginals(pot)
    mg, lz, fl, kern = _marg(pot, dev, None, 0)
    assert kern == "summary_tc_kernel", kern
    check_logz(lz, lz_ref)
    assert (fl == fl_ref).all()
    check_marg(mg, mg_ref)


@pytest.mark.parametrize("B,N,K,C", [(3, 60, 4, 20), (2, 41, 3, 7), (2, 33, 8, 16)])
def test_plan_invariance(dev, B, N, K, C):
    """Segmental kernel (auto at this length) and the expanded chain at L = 1 (Fig. 4 tree),
    L = 5, L = 16 and L = E (serial sweeps of the expanded chain) all match the oracle."""
    pot = _pot(B, N, K, C, N + K + C)
    lengths = np.array([N] + [max(1, N - 7 * i) for i in range(1, B)], np.int32)
    lz_ref, mg_ref, fl_ref = oracle.semimarkov_marginals(pot, lengths)
    kernels = set()
    for L in (0, 1, 5, 16, N - 1):
        mg, lz, fl, kern = _marg(pot, dev, lengths, L)
        kernels.add(kern)
        check_logz(lz, lz_ref)
        assert (fl == fl_ref).all(), (L, fl, fl_ref)
        check_marg(mg, mg_ref)
    assert "semimarkov_kernel" in kernels and len(kernels) >= 2, kernels


def test_expanded_lengths_and_flags(dev):
    B, N, K, C = 7, 30, 4, 6
    pot = _pot(B, N, K, C, 3)
    pot[2] = -np.inf                     # EMPTY
    pot[3, 5, 1, 2, 2] = np.nan          # NONFINITE (a used part)
    pot[5, 5, 3, 0, 0] = np.nan          # segment 5 -> 9 ends beyond len 7: unused, ignored
    lengths = np.array([30, 1, 30, 30, 0, 7, 2], np.int32)
    lz_ref, mg_ref, fl_ref = oracle.semimarkov_marginals(pot, lengths)
    for L in (3, 29):
        mg, lz, fl, _ = _marg(pot, dev, lengths, L)
        check_logz(lz, lz_ref)
        assert (fl == fl_ref).all(), (L, fl, fl_ref)
        check_marg(mg, mg_ref)


@pytest.mark.parametrize("B,N,K,C", [(3, 40, 4, 5), (2, 70, 3, 12)])
def test_expanded_viterbi_bit_exact(dev, B, N, K, C):
    """The max semiring over the expanded chain (serial and chunked Viterbi) reproduces the
    canonical segmentation of reading R18 and its score exactly; coarse values make ties
    frequent."""
    rng = np.random.default_rng(N * C)
    pot = (rng.integers(-3, 4, size=(B, N - 1, K, C, C)) * 0.5).astype(np.float32)
    lengths = np.array([N] + [N - 11 * i for i in range(1, B)], np.int32)
    seg_ref, s_ref, f_ref = oracle.semimarkov_viterbi(pot, lengths)
    lt = torch.from_numpy(lengths).to(dev)
    for L in (0, 1, 6, N - 1):
        tsb.set_plan_chunk(L)
        seg, score, fl = tsb.semimarkov_viterbi(torch.from_numpy(pot).to(dev), lt)
        np.testing.assert_array_equal(fl.cpu().numpy().astype(np.uint32), f_ref, err_msg=f"L={L}")
        np.testing.assert_array_equal(seg.cpu().numpy(), seg_ref, err_msg=f"L={L}")
        ok = f_ref == 0
        assert (score.cpu().numpy()[ok] == s_ref[ok].astype(np.float32)).all(), L
