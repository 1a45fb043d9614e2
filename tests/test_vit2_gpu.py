"""GPU parity of the cluster column-split Viterbi forward (viterbi2.cu, C in {128, 256})
against the fp64 oracle: bit-identical paths, scores and flags for every forced cluster size
G, including coarse dyadic inputs with many exact ties (reading R5: smallest index wins),
ragged lengths, masks and the EMPTY / NONFINITE / BADLEN flags.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2002_00876_b200 as tsb
import tsgen
from _util import check_viterbi

pytestmark = pytest.mark.gpu


def vit_check(pot_np, lengths_np, dev):
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot_np, lengths_np, threads=8)
    pot = torch.from_numpy(np.ascontiguousarray(pot_np)).to(dev)
    lengths = (torch.from_numpy(lengths_np.astype(np.int32)).to(dev)
               if lengths_np is not None else None)
    path, score, flags = tsb.viterbi(pot, lengths)
    check_viterbi(path.cpu().numpy(), score.cpu().numpy(), p_ref, s_ref)
    assert (flags.cpu().numpy().astype(np.uint32) == f_ref).all()
    m, lz, _ = tsb.marginals(pot, lengths, semiring="max")
    np.testing.assert_array_equal(m.cpu().numpy(),
                                  oracle.max_indicator(p_ref, pot_np.shape[-1], lengths_np))


@pytest.fixture
def split():
    yield tsb.set_viterbi_split
    tsb.set_viterbi_split(0)


@pytest.mark.parametrize("C,G", [(256, 1), (256, 2), (256, 4), (256, 8), (128, 1), (128, 2),
                                 (128, 4), (256, 0), (128, 0)])
def test_vit2_shapes(dev, split, C, G):
    split(G)
    for N in (2, 3, 9, 40):
        vit_check(tsgen.potentials(3, N, C, seed=N + C + G), None, dev)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_vit2_ties(dev, split, G):
    # quantum 2^0: integer-valued scores in [-4, 4] -> many equal maxima per column
    split(G)
    vit_check(tsgen.potentials(2, 30, 256, seed=11, s=0), None, dev)
    vit_check(tsgen.potentials(2, 30, 128, seed=12, s=0), None, dev)
    vit_check(np.zeros((2, 6, 256, 256), dtype=np.float32), None, dev)


@pytest.mark.parametrize("G", [2, 4])
def test_vit2_lengths_flags_masks(dev, split, G):
    split(G)
    B, N, C = 7, 25, 256
    pot = tsgen.tagging_potentials(B, N, C, seed=G, mask_frac=0.3)
    lengths = np.array([1, 2, 25, 13, 0, 26, 20], dtype=np.int32)
    pot[2] = -np.inf                  # EMPTY
    pot[3, 4, 200, 7] = np.nan        # NONFINITE
    pot[6, 10, 3, 250] = np.inf       # +inf
    vit_check(pot, lengths, dev)


def test_vit2_matches_legacy_kernel(dev, split):
    pot = torch.from_numpy(tsgen.potentials(5, 64, 256, seed=3)).to(dev)
    split(-1)
    p1, s1, f1 = tsb.viterbi(pot)
    split(2)
    p2, s2, f2 = tsb.viterbi(pot)
    assert torch.equal(p1, p2) and torch.equal(s1, s2) and torch.equal(f1, f2)
