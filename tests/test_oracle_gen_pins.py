"""Pins for the oracle's on-the-fly generator mode and for max_indicator.

`oracle_gen_marginals` / `oracle_gen_viterbi` (oracle/oracle.c) are the checkers of every
full-size GPU parity test (cfg3..cfg5 do not fit a materialised fp64 host copy), so they
are pinned here, without a GPU, against:

  * brute-force enumeration of all C^n labelings (P:149 footnote) on tiny
    generated chains — the definition itself, not another oracle routine;
  * the resident-buffer oracle (`oracle_chain_*`, itself pinned by brute force in
    test_oracle_pins.py) on materialised tsgen potentials at sizes enumeration cannot
    reach, for several (B, N, C, s) and sparse / unsorted / first-and-last edge lists,
    for every sequence b of the batch (so the global index b·E + t is exercised).

A generator-mode indexing slip (E_global = N instead of N-1, a transposed (i, j), a
dropped batch offset) changes the generated l and fails these.  `max_indicator`
(∂A*/∂l) is pinned against finite differences of the brute-force max.
"""
import numpy as np
import pytest

import oracle
import tsgen
from oracle import brute


# ----------------------------------------------------------- brute force, tiny chains

@pytest.mark.parametrize("B,N,C,s", [(3, 5, 3, 15), (2, 4, 4, 9), (4, 6, 2, 3), (2, 1, 4, 15),
                                     (2, 2, 5, 12)])
def test_gen_marginals_equal_enumeration(B, N, C, s):
    seed = 0x5EED + 17 * N + C
    pot = tsgen.potentials(B, N, C, seed, s)  # what the generator mode must regenerate
    for b in range(B):
        edges = list(range(N - 1))
        lz, ed, mg, fl = oracle.gen_marginals(seed, s, b, N, C, edges)
        assert fl == 0
        A = brute.log_partition(pot[b], N)
        assert abs(lz - A) <= 1e-12 * max(1.0, abs(A)), (b, lz, A)
        if edges:
            np.testing.assert_allclose(mg, brute.marginals(pot[b], N), rtol=0, atol=1e-12)


@pytest.mark.parametrize("B,N,C,s", [(3, 5, 3, 0), (2, 6, 3, 1), (4, 4, 4, 0), (2, 1, 3, 0)])
def test_gen_viterbi_equal_enumeration(B, N, C, s):
    # s = 0/1: integer / half-integer potentials, so ties are frequent and the R5 rule counts
    seed = 0xBEEF + 31 * N + C
    pot = tsgen.potentials(B, N, C, seed, s)
    for b in range(B):
        path, score, fl = oracle.gen_viterbi(seed, s, b, N, C)
        z, best = brute.argmax(pot[b], N)
        assert fl == 0
        np.testing.assert_array_equal(path, z)
        assert score == best


# ---------------------------------------- resident-buffer oracle, larger generated chains

GEN_CASES = [
    # (B, N, C, s, edges)  edges: sparse, unsorted, first and last, duplicates-free
    (3, 40, 7, None, [39 - 1, 0, 17, 5]),
    (2, 129, 16, 13, [127, 64, 0, 1, 126]),
    (4, 33, 20, 15, [0, 31, 16]),
    (1, 300, 5, 6, [299 - 1, 150, 0, 149, 151]),
    (2, 2, 9, 15, [0]),
    (3, 17, 3, 2, []),  # logZ only
]


@pytest.mark.parametrize("B,N,C,s,edges", GEN_CASES)
def test_gen_marginals_equal_resident_oracle(B, N, C, s, edges):
    seed = 0x200200876 + 1000 * C + N
    s_eff = tsgen.quantum(N - 1) if s is None else s
    pot = tsgen.potentials(B, N, C, seed, s_eff)
    lz_ref, mg_ref, fl_ref = oracle.chain_marginals(pot)
    for b in range(B):
        lz, ed, mg, fl = oracle.gen_marginals(seed, s_eff, b, N, C, edges)
        assert list(ed) == sorted(edges)
        assert fl == fl_ref[b]
        assert abs(lz - lz_ref[b]) <= 1e-13 * max(1.0, abs(lz_ref[b])), (b, lz, lz_ref[b])
        for k, e in enumerate(ed):
            np.testing.assert_allclose(mg[k], mg_ref[b, e], rtol=0, atol=1e-14)
            # and the per-edge normalisation the definition fixes (Σ μ_t = 1)
            assert abs(mg[k].sum() - 1.0) < 1e-12


@pytest.mark.parametrize("B,N,C,s", [(3, 40, 7, 0), (2, 129, 16, 13), (2, 64, 33, 1),
                                     (1, 300, 5, 0), (3, 1, 4, 15)])
def test_gen_viterbi_equal_resident_oracle(B, N, C, s):
    seed = 0x200200876 + 77 * C + N
    pot = tsgen.potentials(B, N, C, seed, s)
    p_ref, s_ref, f_ref = oracle.chain_viterbi(pot)
    for b in range(B):
        path, score, fl = oracle.gen_viterbi(seed, s, b, N, C)
        np.testing.assert_array_equal(path, p_ref[b])
        assert score == s_ref[b] and fl == f_ref[b]


def test_gen_mode_reads_the_sequence_it_is_asked_for():
    # sequences differ, so an ignored or mis-scaled b would repeat sequence 0
    seed, N, C, s = 12345, 30, 6, 15
    a = [oracle.gen_marginals(seed, s, b, N, C, [])[0] for b in range(4)]
    assert len(set(a)) == 4
    pot = tsgen.potentials(4, N, C, seed, s)
    for b in range(4):
        assert abs(a[b] - brute_free_logz(pot[b])) < 1e-12 * abs(a[b])


def brute_free_logz(pot_seq):
    """log Z by the plain matrix-product definition in linear space: small
    |l| <= 4 and short chains keep exp() in range, so no stabilisation is needed."""
    M = np.exp(pot_seq.astype(np.float64))
    v = np.ones(M.shape[1])
    for t in range(M.shape[0]):
        v = v @ M[t]
    return float(np.log(v.sum()))


# --------------------------------------------------------------------- max_indicator

@pytest.mark.parametrize("seed", range(6))
def test_max_indicator_is_the_derivative_of_the_brute_force_max(seed):
    # A*(l) = max_z Score(z) is piecewise linear; where the maximiser is unique,
    # dA*/dl_p = [p on z*].  Continuous random l makes it unique a.s.
    rng = np.random.default_rng(seed)
    B, N, C = 2, 5, 3
    lengths = np.array([N, 3], dtype=np.int32)
    pot = rng.normal(size=(B, N - 1, C, C)).astype(np.float32)
    path, _, _ = oracle.chain_viterbi(pot, lengths)
    ind = oracle.max_indicator(path, C, lengths)
    h = 1e-3
    for b in range(B):
        n = int(lengths[b])
        base = brute.argmax(pot[b], n)[1]
        for t in range(N - 1):
            for i in range(C):
                for j in range(C):
                    q = pot[b].astype(np.float64).copy()
                    q[t, i, j] += h
                    d = (brute.argmax(q, n)[1] - base) / h
                    assert abs(d - ind[b, t, i, j]) < 1e-6, (b, t, i, j, d)
    assert ind[1, 2:].sum() == 0  # edges beyond len 3 carry no indicator
