"""GPU parity of K-best Viterbi (Table 2 'K-Max') through the C ABI
against the fp64 oracle (oracle.chain_kbest, pinned against sorted enumeration): paths
and scores bit-identical (dyadic inputs), order = score desc then reverse-lexicographic
(R16), flags identical."""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen

pytestmark = pytest.mark.gpu


def _coarse(B, N, C, seed):
    return (np.random.default_rng(seed).integers(-2, 3, size=(B, N - 1, C, C)) * 0.5
            ).astype(np.float32)


@pytest.fixture(autouse=True, params=[0, 1, 2, 8])
def _split(request):
    """Every case under the automatic lanes-per-column choice and forced S = 1, 2, 8."""
    tsb.set_kbest_split(request.param)
    yield
    tsb.set_kbest_split(0)


def _check(pot, K, dev, lengths=None):
    p_ref, s_ref, f_ref = oracle.chain_kbest(pot, K, lengths)
    lt = torch.from_numpy(lengths).to(dev) if lengths is not None else None
    paths, scores, flags = tsb.kbest(torch.from_numpy(pot).to(dev), K, lt)
    np.testing.assert_array_equal(paths.cpu().numpy(), p_ref)
    s = scores.cpu().numpy()
    r = s_ref.astype(np.float32)
    assert ((s == r) | (np.isnan(s) & np.isnan(r))).all(), (s, r)
    assert (flags.cpu().numpy().astype(np.uint32) == f_ref).all()


@pytest.mark.parametrize("B,N,C,K", [(2, 6, 3, 5), (3, 25, 20, 8), (2, 12, 64, 16),
                                     (2, 30, 7, 3), (1, 5, 256, 4), (2, 9, 128, 2),
                                     (3, 4, 2, 16), (2, 40, 20, 1)])
def test_kbest_ties(dev, B, N, C, K):
    _check(_coarse(B, N, C, N * C + K), K, dev)


@pytest.mark.parametrize("K", [1, 4, 16])
def test_kbest_generator_inputs(dev, K):
    _check(tsgen.potentials(3, 25, 20, seed=7 + K), K, dev)


def test_kbest_k1_equals_viterbi(dev):
    pot = tsgen.potentials(4, 60, 32, seed=3)
    paths, scores, _ = tsb.kbest(torch.from_numpy(pot).to(dev), 1)
    path, score, _ = tsb.viterbi(torch.from_numpy(pot).to(dev))
    assert torch.equal(paths[:, 0], path) and torch.equal(scores[:, 0], score)


def test_kbest_lengths_flags_short(dev):
    B, N, C = 6, 7, 3
    pot = _coarse(B, N, C, 1)
    pot[2] = -np.inf                       # EMPTY
    pot[3, 2, 1, 1] = np.nan               # NONFINITE
    lengths = np.array([7, 1, 7, 7, 0, 2], np.int32)   # len 1, BADLEN, len 2 (9 labelings)
    _check(pot, 12, dev, lengths)


@pytest.mark.parametrize("C,K", [(20, 8), (64, 4), (128, 16), (5, 16)])
def test_kbest_sparse_support(dev, C, K):
    """Most transitions -inf (a banded, partly masked support): columns often have fewer than
    KM finite heads, so the step's pruning bound T (the KM-th largest head) is -inf and only
    the finite candidates may enter; plus coarse ties on the finite entries."""
    B, N = 3, 33
    rng = np.random.default_rng(C * 7 + K)
    pot = (rng.integers(-2, 3, size=(B, N - 1, C, C)) * 0.5).astype(np.float32)
    i, j = np.meshgrid(np.arange(C), np.arange(C), indexing="ij")
    band = np.abs(i - j) <= 1
    pot[:, :, ~band] = -np.inf
    pot[rng.random(pot.shape) < 0.3] = -np.inf
    _check(pot, K, dev)
